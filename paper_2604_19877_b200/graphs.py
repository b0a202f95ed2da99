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
    """Construction runs `warmup` eager decode steps (first-launch module loading and kernel
    attributes happen outside the capture), then captures one step.  The warm-up advances the
    engine's state: by default the engine is reset afterwards (build graphs on an empty engine,
    before prefill); preserve_state=True instead snapshots and restores exactly what a decode
    step writes — the lengths, the KV slots of the warm-up positions and the GDN/KDA states and
    conv rings (the recurrent states are rewritten whole, so they are copied whole)."""

    def __init__(self, model, feedback: bool = False, warmup: int = 2, preserve_state: bool = False):
        self.model = model
        self.feedback = feedback
        self.graph = torch.cuda.CUDAGraph()
        # the snapshot copies are enqueued on the current stream BEFORE the side stream is told
        # to wait for it: the warm-up steps below must not start while the copies still read
        saved = self._snapshot(warmup) if preserve_state else None
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(warmup):
                model.decode_body()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        if saved is not None:
            self._restore(saved)
        elif warmup:
            model.reset()
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

    def _kv_index(self, kind, steps):
        """(page, offset) of the KV slots `steps` decode steps write, per sequence."""
        from .placement import SWA
        m = self.model
        P = m.cfg.page_size
        pos = m.seq_lens.long()[:, None] + torch.arange(max(steps, 1), device=m.device)[None]
        if kind == SWA:
            slot, bt = pos % m.cfg.window, m.swa_block_table
        else:
            slot, bt = pos.clamp(max=m.max_len - 1), m.fa_block_table
        page = torch.gather(bt.long(), 1, (slot // P).clamp(max=bt.shape[1] - 1))
        return page.reshape(-1), (slot % P).reshape(-1)

    def _snapshot(self, steps):
        from .placement import FA, SWA
        m = self.model
        snap = {"seq_lens": m.seq_lens.clone(), "layers": []}
        for kind, st in zip(m.kinds, m.state):
            if kind in (FA, SWA):
                page, off = self._kv_index(kind, steps)
                snap["layers"].append(("kv", page, off, st["k"][page, :, off].clone(), st["v"][page, :, off].clone()))
            else:
                snap["layers"].append(("rec", {k: v.clone() for k, v in st.items()}))
        return snap

    def _restore(self, snap):
        m = self.model
        m.seq_lens.copy_(snap["seq_lens"])
        for st, rec in zip(m.state, snap["layers"]):
            if rec[0] == "kv":
                _, page, off, k, v = rec
                st["k"][page, :, off] = k
                st["v"][page, :, off] = v
            else:
                for k, v in rec[1].items():
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
