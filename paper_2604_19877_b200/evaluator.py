"""Trace log-likelihood placement scorer for the reference's search loop.

The paper scores placements by the log-likelihood of fixed teacher traces under each
candidate placement, normalised by the number of completion tokens (R/PAPER.md:917-921,
1939) and optionally min-max normalised over random placements (R/PAPER.md:921).  The
reference consumes such scores through its line protocol (`SubprocessEvaluator`,
R/pkg/src/placeopt/acquisition.py:312-340): placement codes on stdin, one per line, one
float per line on stdout, non-zero exit on failure.  This module is that evaluator:

    placeopt explore --evaluator "subprocess:python -m paper_2604_19877_b200.evaluator --config apriel" ...

Every placement is a prefill-only forward of the traces through the runtime's own kernels,
on one resident supernet (serving.SupernetStore): the shared trunk is loaded once, each
(layer, mixer) weight set on first use.  There are no checkpoints or teacher traces
offline, so the weights are the seeded random init and the traces are seeded synthetic
token sequences unless --traces gives an int tensor file [N, T].
"""
from __future__ import annotations

import argparse
import sys

import torch

from .config import CONFIGS
from .placement import DEFAULT_CATALOG, Placement


def loglik_from_logits(logits: torch.Tensor, tokens: torch.Tensor, prompt_len: int = 1) -> torch.Tensor:
    """Per-sequence mean log-likelihood of the completion tokens tokens[:, prompt_len:] (each
    predicted by the logits of the position before it; logits [B, T, V]).  prompt_len = 1
    scores every next-token position."""
    B, T, _ = logits.shape
    if not 1 <= prompt_len < T:
        raise ValueError(f"prompt_len {prompt_len} must be in [1, {T})")
    out = torch.empty(B, dtype=torch.float64)
    for b in range(B):  # one row at a time: [T, V] fp32 log-softmax, not [B, T, V]
        lp = torch.log_softmax(logits[b, prompt_len - 1:-1].float(), dim=-1)
        tgt = tokens[b, prompt_len:].to(device=lp.device, dtype=torch.long)
        out[b] = lp.gather(-1, tgt[:, None]).double().mean().item()
    return out


def trace_loglik(model, traces: torch.Tensor, prompt_len: int = 1) -> float:
    """Mean completion-token log-likelihood of traces [N, T] (N a multiple of model.B) under the
    model's placement, normalised by completion tokens (R/PAPER.md:917-921)."""
    N = traces.shape[0]
    if N % model.B:
        raise ValueError(f"{N} traces is not a multiple of the engine batch {model.B}")
    total = 0.0
    for i in range(0, N, model.B):
        toks = traces[i:i + model.B]
        logits = model.prefill(toks, return_all=True)
        total += float(loglik_from_logits(logits, toks, prompt_len).sum())
    return total / N


def parse_placements(lines, num_layers: int) -> list[str]:
    """Validate every input line first (before any GPU work): unknown codes or a wrong layer
    count fail the whole call, as the reference's protocol expects (EvaluatorError)."""
    codes = []
    for n, line in enumerate(lines, start=1):
        code = line.strip()
        if not code:
            continue
        try:
            p = Placement.from_codes(code, DEFAULT_CATALOG)
        except ValueError as exc:
            raise ValueError(f"line {n}: {exc}") from exc
        if len(p.assignments) != num_layers:
            raise ValueError(f"line {n}: placement has {len(p.assignments)} layers, expected {num_layers}")
        codes.append(code)
    return codes


def synthetic_traces(n: int, length: int, vocab: int, seed: int) -> torch.Tensor:
    return torch.randint(0, vocab, (n, length), generator=torch.Generator().manual_seed(seed), dtype=torch.int64)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--config", default="tiny", choices=sorted(CONFIGS))
    ap.add_argument("--traces", default="", help="torch int tensor file [N, T]; default: synthetic")
    ap.add_argument("--num-traces", type=int, default=4)
    ap.add_argument("--trace-len", type=int, default=256)
    ap.add_argument("--batch", type=int, default=4, help="traces per prefill")
    ap.add_argument("--seed", type=int, default=0, help="weight seed")
    ap.add_argument("--init-device", default="cuda", help="where the seeded weight draws run (cpu = the oracle's weights)")
    ap.add_argument("--trace-seed", type=int, default=1)
    ap.add_argument("--prompt-len", type=int, default=1,
                    help="tokens of each trace that are prompt: only the completion after them is scored")
    ap.add_argument("--normalize", default="", help="lo,hi: print (ll - lo) / (hi - lo) (R/PAPER.md:921)")
    a = ap.parse_args(argv)
    cfg = CONFIGS[a.config]
    try:
        codes = parse_placements(sys.stdin.read().splitlines(), cfg.num_layers)
    except ValueError as exc:
        print(f"evaluator: {exc}", file=sys.stderr)
        return 2
    traces = torch.load(a.traces) if a.traces else synthetic_traces(a.num_traces, a.trace_len, cfg.vocab,
                                                                     a.trace_seed)
    traces = torch.as_tensor(traces, dtype=torch.int64)
    lo_hi = [float(x) for x in a.normalize.split(",")] if a.normalize else None
    from . import ops
    from .model import Supernet
    from .serving import SupernetStore
    store = SupernetStore(cfg, seed=a.seed, init_device=a.init_device)
    B = min(a.batch, traces.shape[0])
    block = ops.gemm_swiglu_block(cfg.ffn)  # the FFN decode layout, shared by every placement
    N = traces.shape[0]
    for code in codes:
        # every trace is scored: full batches of B, then one engine for the remainder
        total = 0.0
        for b, lo, hi in ((B, 0, N // B * B), (N % B, N // B * B, N)):
            if hi > lo:
                model = Supernet(cfg, code, batch=b, max_len=traces.shape[1],
                                 weights=store.weights(code, swiglu_block=block))
                total += trace_loglik(model, traces[lo:hi], a.prompt_len) * (hi - lo)
                del model
        ll = total / N
        if lo_hi:
            ll = (ll - lo_hi[0]) / (lo_hi[1] - lo_hi[0])
        print(repr(float(ll)), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
