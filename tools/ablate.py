"""Marginal in-graph cost of each kernel class of the decode step: re-capture the graph with
one class replaced by a no-op (results are wrong; only the timing is read) and report
base - ablated.  Unlike tools/step_breakdown.py this keeps PDL overlap intact, so it shows
what removing / speeding up a kernel class would actually buy.

  python tools/ablate.py [--preset ... --batch 64 --context 32768] [--only norm,rope]
"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import fill_synthetic  # noqa: E402
from paper_2604_19877_b200 import APRIEL, PRESETS, ops  # noqa: E402
from paper_2604_19877_b200.graphs import DecodeGraph  # noqa: E402
from paper_2604_19877_b200.model import Supernet  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--preset", default="Reg|Lklhd-10")
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--context", type=int, default=32768)
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--only", default="")
a = ap.parse_args()


def noop(*args, **kw):
    return None


_gemm = ops.gemm_decode


def gemm_skip_if(pred):
    def f(x, w, out, mode):
        if pred(x, w, out, mode):
            return 1
        return _gemm(x, w, out, mode)
    return f


c = APRIEL
ABL = {
    "in_proj": [(ops, "gemm_decode", gemm_skip_if(lambda x, w, o, m: m == "store" and x.shape[1] == c.hidden
                                                  and o.shape[-1] in (c.gdn_in_width, c.kda_in_width))),
                (ops, "gemm_decode_attn_in", noop)],
    "out_proj": [(ops, "gemm_decode", gemm_skip_if(lambda x, w, o, m: m == "partial" and x.shape[1] != c.ffn))],
    "ffn_down": [(ops, "gemm_decode", gemm_skip_if(lambda x, w, o, m: m == "partial" and x.shape[1] == c.ffn))],
    "ffn_gate_up": [(ops, "gemm_decode", gemm_skip_if(lambda x, w, o, m: m == "swiglu_il"))],
    "lm_head": [(ops, "gemm_decode", gemm_skip_if(lambda x, w, o, m: o.shape[-1] == c.vocab))],
    "kda_gates": [(ops, "kda_gate_factors", noop)],
    "norm": [(ops, "add_rmsnorm", noop)],
    "gdn": [(ops, "gdn_decode", noop)],
    "kda": [(ops, "kda_decode", noop)],
    "attn": [(ops, "attn_decode", noop)],
}

m = Supernet(APRIEL, PRESETS[a.preset].layer_string, batch=a.batch, max_len=a.context + 256, dtype=torch.bfloat16)


def step_ms():
    g = DecodeGraph(m, feedback=False)
    fill_synthetic(m, a.context)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.steps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / a.steps)
    del g
    return best


base = step_ms()
print(f"base {base:.3f} ms/step")
names = [n for n in ABL if not a.only or n in a.only.split(",")]
for n in names:
    saved = [(mod, attr, getattr(mod, attr)) for mod, attr, _ in ABL[n]]
    for mod, attr, f in ABL[n]:
        setattr(mod, attr, f)
    try:
        t = step_ms()
    finally:
        for mod, attr, f in saved:
            setattr(mod, attr, f)
    print(f"without {n:10s} {t:.3f} ms/step  marginal cost {base - t:7.3f} ms")
