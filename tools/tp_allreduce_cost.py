"""Per-layer cost of the head-parallel decode all-reduce fused into add+RMSNorm
(csrc/sn_tp.cu) at Apriel shapes, on ONE GPU: the "peer" slab buffers and arrival counters
are local allocations (counters already satisfied), so this measures the kernel's own
cost — reading world x S fp32 slabs per row, summing in rank order, the norm — without the
NVLink transfer latency a multi-GPU node adds.  Baseline: the single-GPU sn_add_rmsnorm over
the same S slabs.  CUDA graph of 48 x 2 launches (two norms per layer), events.

  python tools/tp_allreduce_cost.py [--batch 64]
"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_19877_b200 import APRIEL, ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--splits", type=int, default=4)
a = ap.parse_args()
B, d, S, L = a.batch, APRIEL.hidden, a.splits, 48


def graph_time(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=s):
        for _ in range(2 * L):
            fn()
    g.replay()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / (2 * L) * 1e3)
    return best


resid = torch.randn(B, d, device="cuda")
w = torch.ones(d, device="cuda", dtype=torch.bfloat16)
out = torch.empty(B, d, device="cuda", dtype=torch.bfloat16)
slabs = torch.randn(S, B, d, device="cuda") * 1e-3
base = graph_time(lambda: ops.add_rmsnorm(None, resid, w, out, 1e-5, partials=slabs, nsplit=S))
print(f"B={B} d={d} S={S}: add+RMSNorm over local slabs (TP=1)             {base:6.2f} us/launch")
for world in (2, 4, 8):
    peers = [torch.randn(S, B, d, device="cuda") * 1e-3 for _ in range(world)]
    ctr = [torch.zeros(4, device="cuda", dtype=torch.int32) for _ in range(world)]
    slab_ptrs = torch.tensor([p.data_ptr() for p in peers], dtype=torch.int64, device="cuda")
    ctr_ptrs = torch.tensor([c.data_ptr() for c in ctr], dtype=torch.int64, device="cuda")
    t = graph_time(lambda: ops.tp_allreduce_add_rmsnorm(slab_ptrs, ctr_ptrs, world, 0, S, resid,
                                                        w, out, 1e-5))
    print(f"B={B} d={d} S={S}: fused all-reduce + add+RMSNorm, world {world} (local peers) {t:6.2f} us/launch"
          f"  (+{t - base:5.2f} us; {world * S * B * d * 4 / t / 1e3:6.0f} GB/s of slab reads)")
