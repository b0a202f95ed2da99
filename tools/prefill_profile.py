"""Where does prefill time go?  One Apriel-48 prefill of B x T tokens (random-init weights),
timed with CUDA events, then the same call under torch.profiler for a per-kernel table.

  python tools/prefill_profile.py --preset 'Reg|Lklhd-10' --batch 1 --tokens 16384
"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_19877_b200 import APRIEL, PRESETS  # noqa: E402
from paper_2604_19877_b200.model import Supernet  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--preset", default="Reg|Lklhd-10")
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--tokens", type=int, default=16384)
ap.add_argument("--top", type=int, default=25)
a = ap.parse_args()
m = Supernet(APRIEL, PRESETS[a.preset].layer_string, batch=a.batch, max_len=a.tokens + 64, dtype=torch.bfloat16)
toks = torch.randint(0, APRIEL.vocab, (a.batch, a.tokens), generator=torch.Generator().manual_seed(1))
m.prefill(toks)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
m.reset()
e0.record()
m.prefill(toks)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
ntok = a.batch * a.tokens
print(f"prefill {a.preset} B={a.batch} T={a.tokens}: {ms:.1f} ms  {ntok / ms * 1e3:.0f} tok/s")
m.reset()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    m.prefill(toks)
    torch.cuda.synchronize()
tot = {}
for ev in prof.key_averages():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        tot[ev.key] = (getattr(ev, "device_time_total", 0) or getattr(ev, "cuda_time_total", 0), ev.count)
s = sum(v[0] for v in tot.values())
print(f"kernel time {s / 1e3:.1f} ms")
for k, (t, n) in sorted(tot.items(), key=lambda kv: -kv[1][0])[: a.top]:
    print(f"{t / 1e3:9.2f} ms {t / s * 100:5.1f}%  x{n:4d}  {k[:100]}")
