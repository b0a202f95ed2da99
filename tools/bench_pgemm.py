"""Prefill GEMM throughput (tcgen05 sn_gemm_prefill vs cuBLAS torch.mm) on the Apriel prefill
projection shapes at a 16K-token prompt; CUDA events, best of 5 after warm-up."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_19877_b200 import APRIEL, ops  # noqa: E402

c = APRIEL
M = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
h = ops.gemm_swiglu_block(c.ffn)
shapes = [("gdn_in", c.gdn_in_width, c.hidden), ("attn_qkv", c.attn_qkv_width, c.hidden),
          ("o_proj", c.hidden, c.gdn_value_dim), ("ffn_gate_up", 2 * c.ffn, c.hidden), ("ffn_down", c.hidden, c.ffn)]


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


a = torch.randn(M, max(c.ffn, c.hidden), device="cuda").to(torch.bfloat16)
for name, N, K in shapes:
    x = a[:, :K].contiguous()
    w = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
    fl = 2.0 * M * N * K
    t_cub = timeit(lambda: torch.mm(x, w.t()))
    if name == "ffn_gate_up":
        wil = ops.interleave_swiglu(w, h)
        out = torch.empty(M, c.ffn, device="cuda", dtype=torch.bfloat16)
        t_own = timeit(lambda: ops.gemm_prefill(x, wil, out, swiglu_h=h))
    else:
        out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        t_own = timeit(lambda: ops.gemm_prefill(x, w, out))
    print(f"{name:12s} M={M} N={N} K={K}: ours {t_own:7.3f} ms {fl / t_own / 1e9:7.1f} TFLOP/s | "
          f"cuBLAS {t_cub:7.3f} ms {fl / t_cub / 1e9:7.1f} TFLOP/s | ratio {t_cub / t_own:.2f}")
