"""Per-CTA timeline of one fused decode chain inside the graphed Apriel decode step
(csrc/sn_chain.cu %globaltimer stamps, sn_decode_chain_trace).

For each phase of the traced chain: when its inputs were released to the producer (barrier
or the previous kernel), when each CTA finished its part (epilogue / norm rows) and arrived,
and for the barrier after it the last arrival vs the first release (propagation).

  python tools/chain_trace.py [--sites 5,20] [--batch 64 --context 32768]
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
from paper_2604_19877_b200.placement import layer_kinds  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--preset", default="Reg|Lklhd-10")
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--context", type=int, default=32768)
ap.add_argument("--sites", default="5,14,20")
a = ap.parse_args()

lib = ops._lib.load()
cfg = APRIEL
kinds = layer_kinds(PRESETS[a.preset].layer_string)
model = Supernet(cfg, PRESETS[a.preset].layer_string, batch=a.batch, max_len=a.context + 64, dtype=torch.bfloat16,
                 fused_chain=True)
base_graph = DecodeGraph(model, feedback=True)  # warm-up on the empty engine (it resets)
fill_synthetic(model, a.context)
names = "ASKG"
for site in [int(x) for x in a.sites.split(",")]:
    buf = torch.zeros(148, 40, dtype=torch.int64, device="cuda")
    orig = model._chain
    seen = {}

    def traced(s, phases, orig=orig, site=site):
        if s == site:
            lib.sn_decode_chain_trace(ctypes_ptr(buf))
            seen["phases"] = [("G" if p["kind"] == 0 else "N") + (f"/m{p['mode']}" if p["kind"] == 0 else "")
                              for p in phases]
        orig(s, phases)
        if s == site:
            lib.sn_decode_chain_trace(None)

    def ctypes_ptr(t):
        import ctypes
        return ctypes.c_void_p(t.data_ptr())

    model._chain = traced
    g = DecodeGraph(model, feedback=True, preserve_state=True, warmup=0)
    model._chain = orig
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    t = buf.cpu().double()
    used = t[:, 0] > 0
    t = t[used]
    t0 = t[:, 0].min()
    us = lambda x: (x - t0) / 1e3
    prev_kind = kinds[site - 1] if site > 0 else None
    next_kind = kinds[site] if site < len(kinds) else None
    print(f"site {site} (after layer {site - 1} {names[prev_kind] if prev_kind is not None else '-'}, "
          f"before layer {site} {names[next_kind] if next_kind is not None else '-'}), {int(used.sum())} CTAs, "
          f"kernel {us(t[:, 1].max()):.1f} us (start spread {us(t[:, 0].max()):.1f})")
    for p, nm in enumerate(seen["phases"]):
        rel, done, arr, nrel = (t[:, 2 + 4 * p], t[:, 3 + 4 * p], t[:, 4 + 4 * p], t[:, 5 + 4 * p])
        def stat(x):
            x = x[x > 0]
            if x.numel() == 0:
                return "      -      "
            return f"{us(x.min()):6.1f}/{us(x.median()):6.1f}/{us(x.max()):6.1f}"
        print(f"  phase {p} {nm:7s} inputs-ready {stat(rel)}  norm-release {stat(nrel)}  done {stat(done)}  "
              f"arrived {stat(arr)}")
    del g
