"""In-graph per-kernel time breakdown of one decode step (CUDA events around every launch,
captured as graph event nodes; PDL overlap is lost at the event boundaries, so the sum is an
upper bound of the real step)."""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import fill_synthetic  # noqa: E402
from paper_2604_19877_b200 import APRIEL, PRESETS  # noqa: E402
from paper_2604_19877_b200.graphs import DecodeGraph  # noqa: E402
from paper_2604_19877_b200.model import KernelProbe, Supernet  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--preset", default="Reg|Lklhd-10")
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--context", type=int, default=32768)
ap.add_argument("--steps", type=int, default=10)
a = ap.parse_args()
m = Supernet(APRIEL, PRESETS[a.preset].layer_string, batch=a.batch, max_len=a.context + 128, dtype=torch.bfloat16)
g = DecodeGraph(m, feedback=True, preserve_state=False)  # warm-up + capture on the empty engine (it resets)
fill_synthetic(m, a.context)  # then the KV pools / states at the context length
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.steps):
    g.replay()
e1.record()
torch.cuda.synchronize()
step_ms = e0.elapsed_time(e1) / a.steps
m.probe = KernelProbe(fine=True)
pg = DecodeGraph(m, feedback=True, preserve_state=False, warmup=0)
probe, m.probe = m.probe, None
acc = {}
for _ in range(a.steps):
    pg.replay()
    torch.cuda.synchronize()
    for n, v in probe.collect().items():
        acc.setdefault(n, []).extend(v)
tot = sum(sum(v) for v in acc.values()) / a.steps
print(f"graph step {step_ms:.3f} ms; instrumented sum {tot:.3f} ms")
for n, v in sorted(acc.items(), key=lambda kv: -sum(kv[1])):
    per_step = sum(v) / a.steps
    print(f"{n:22s} {len(v)//a.steps:4d} launches  {per_step*1e3:8.1f} us/step  {per_step/step_ms*100:5.1f}%  {sum(v)/len(v)*1e3:7.2f} us/launch")
