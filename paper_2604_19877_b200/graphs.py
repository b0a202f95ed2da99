"""CUDA graphs per placement (R/PAPER.md:831, 863: "CUDA graphs are pre-captured
for allowed placements, and at runtime the model runner selects the correct
graph").

A decode step is ~10 launches per layer (≈500 for 48 layers); replaying one
captured graph per (placement, batch) removes the per-launch host cost.  Every
kernel reads lengths/positions from device buffers, so one capture serves every
later step.  `feedback=True` appends a device copy next_tokens -> step_tokens so
K replays run K greedy steps with no host round trip; the end-to-end path
(`step_host`) instead copies the step's tokens in from pinned host memory and
the sampled tokens back out, every step.
"""
from __future__ import annotations

import torch


class DecodeGraph:
    def __init__(self, model, feedback: bool = False, warmup: int = 2, preserve_state: bool = True):
        self.model = model
        self.feedback = feedback
        self.graph = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        # warm up on the side stream (cuBLAS handles / workspaces get created outside capture);
        # the state is snapshotted and restored so capture has no visible side effects.
        saved = self._snapshot() if preserve_state else None
        with torch.cuda.stream(s):
            for _ in range(warmup):
                model.decode_body()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        if saved is not None:
            self._restore(saved)
        torch.cuda.synchronize()
        with torch.cuda.graph(self.graph, stream=s):
            model.decode_body()
            if feedback:
                model.step_tokens.copy_(model.next_tokens)
        torch.cuda.synchronize()
        if saved is not None:
            self._restore(saved)  # capture does not execute, but keep the contract explicit
        self._pin_in = torch.empty(model.B, dtype=torch.int32, pin_memory=True)
        self._pin_out = torch.empty(model.B, dtype=torch.int32, pin_memory=True)

    def _snapshot(self):
        m = self.model
        return {"seq_lens": m.seq_lens.clone(), "state": [{k: v.clone() for k, v in st.items()} for st in m.state]}

    def _restore(self, snap):
        m = self.model
        m.seq_lens.copy_(snap["seq_lens"])
        for st, sv in zip(m.state, snap["state"]):
            for k, v in sv.items():
                st[k].copy_(v)

    def replay(self):
        self.graph.replay()

    def step_host(self, tokens_host):
        """End-to-end step through the public API: host tokens in, host tokens out."""
        m = self.model
        self._pin_in.copy_(torch.as_tensor(tokens_host, dtype=torch.int32))
        m.step_tokens.copy_(self._pin_in, non_blocking=True)
        self.graph.replay()
        self._pin_out.copy_(m.next_tokens, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return self._pin_out
