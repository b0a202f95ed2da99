"""Profile one decode step of a preset under ncu (profiling window = one graph replay).

  ncu --profile-from-start off ... python tools/profile_step.py --preset 'Reg|Lklhd-10' --batch 64 --context 32768
"""
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
ap.add_argument("--replays", type=int, default=1)
ap.add_argument("--eager", action="store_true")
ap.add_argument("--chain", action="store_true", help="the opt-in fused decode chains")
a = ap.parse_args()
m = Supernet(APRIEL, PRESETS[a.preset].layer_string, batch=a.batch, max_len=a.context + 64, dtype=torch.bfloat16,
             fused_chain=a.chain)
g = DecodeGraph(m, feedback=True, preserve_state=False)  # warm-up + capture on the empty engine (it resets)
fill_synthetic(m, a.context)  # then the KV pools / states at the context length
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for _ in range(a.replays):
    if a.eager:
        m.decode_body()
    else:
        g.replay()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("profiled", a.replays, "step(s)")
