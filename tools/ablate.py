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
from paper_2604_19877_b200 import model as model_mod  # noqa: E402
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


def gemm_noop_roles(roles):
    def f(x, w, out, mode="store"):
        if mode == "partial":
            return ops.gemm_decode_splits(x.shape[0], out.shape[-1], x.shape[1], "partial")
        return None
    return f


def gemm_skip_if(pred):
    def f(x, w, out, mode="store"):
        if pred(x, w, mode):
            return ops.gemm_decode_splits(x.shape[0], out.shape[-1], x.shape[1], "partial") if mode == "partial" else None
        return _gemm(x, w, out, mode)
    return f


ABL = {
    "ffn_down": [(ops, "gemm_decode", gemm_skip_if(lambda x, w, m: m == "partial" and x.shape[1] == APRIEL.ffn))],
    "ffn_gate_up": [(ops, "gemm_decode", gemm_skip_if(lambda x, w, m: m == "swiglu_il"))],
    "norm": [(ops, "add_rmsnorm", noop)],
    "rope": [(ops, "rope_kv_append", noop)],
    "gdn": [(ops, "gdn_decode", noop)],
    "kda": [(ops, "kda_decode", noop)],
    "attn": [(ops, "attn_decode", noop)],
    "sn_gemm": [(ops, "gemm_decode", gemm_noop_roles(None))],
    "cublas_mm": [(torch, "mm", lambda *a, **k: None), (torch, "bmm", lambda *a, **k: None)],
}

m = Supernet(APRIEL, PRESETS[a.preset].layer_string, batch=a.batch, max_len=a.context + 256, dtype=torch.bfloat16)
fill_synthetic(m, a.context)


def step_ms():
    g = DecodeGraph(m, feedback=False, preserve_state=False)
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
