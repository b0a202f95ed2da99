"""Prefill add + RMSNorm (sn_add_rmsnorm, rows > 512: one CTA per row) at Apriel width:
residual fp32 += delta bf16, out bf16 = RMSNorm(residual) * w.  CUDA events, back-to-back
launches on rotating buffers; algorithmic bytes = 2 x fp32 residual + bf16 delta + bf16 out."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_19877_b200 import ops  # noqa: E402

d = 5120
for rows in (2048, 16384):
    L = 4
    res = [torch.randn(rows, d, device="cuda") for _ in range(L)]
    dl = [torch.randn(rows, d, device="cuda").to(torch.bfloat16) for _ in range(L)]
    out = [torch.empty(rows, d, device="cuda", dtype=torch.bfloat16) for _ in range(L)]
    w = torch.ones(d, device="cuda", dtype=torch.bfloat16)
    for i in range(L):
        ops.add_rmsnorm(dl[i], res[i], w, out[i], 1e-5)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(L):
            ops.add_rmsnorm(dl[i], res[i], w, out[i], 1e-5)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / L)
    nbytes = rows * d * (4 + 4 + 2 + 2)
    print(f"add_rmsnorm rows={rows} d={d}: {best * 1e3:8.1f} us  {nbytes / best / 1e6:6.0f} GB/s")
