"""Decode-step time (graph replay, inputs resident) for one preset — quick A/B of env knobs
(e.g. SN_DECODE_GEMMS) without the full bench.py legs."""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import fill_synthetic  # noqa: E402
from paper_2604_19877_b200 import APRIEL, PRESETS  # noqa: E402
from paper_2604_19877_b200.graphs import DecodeGraph  # noqa: E402
from paper_2604_19877_b200.model import Supernet  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--preset", default="Reg|Lklhd-10")
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--context", type=int, default=32768)
ap.add_argument("--steps", type=int, default=30)
a = ap.parse_args()
m = Supernet(APRIEL, PRESETS[a.preset].layer_string, batch=a.batch, max_len=a.context + 128, dtype=torch.bfloat16,
             fused_chain=bool(os.environ.get("SN_CHAIN")))  # A/B: fused decode chains
g = DecodeGraph(m, feedback=True, preserve_state=False)  # warm-up + capture on the empty engine (it resets)
fill_synthetic(m, a.context)  # then fill the KV / states to the context
for _ in range(5):
    g.replay()
torch.cuda.synchronize()
best = []
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    best.append(e0.elapsed_time(e1) / a.steps)
ms = min(best)
print(f"{'fused chains' if m.use_chain else 'separate kernels'}: {ms:.3f} ms/step "
      f"{a.batch / ms * 1e3:.0f} tok/s  (reps {', '.join(f'{b:.3f}' for b in best)})")
