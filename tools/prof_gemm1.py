"""Single decode-GEMM launch for ncu source-level analysis: python tools/prof_gemm1.py N K mode."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_19877_b200 import ops  # noqa: E402

N, K = int(sys.argv[1]), int(sys.argv[2])
mode = sys.argv[3] if len(sys.argv) > 3 else "store"
M = 64
w = torch.randn(2 * N if mode == "swiglu" else N, K, device="cuda").to(torch.bfloat16)
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
out = torch.zeros(8 if mode == "partial" else 1, M, N, device="cuda",
                  dtype=torch.float32 if mode in ("resid", "partial") else torch.bfloat16)
if mode != "partial":
    out = out[0]
ops.gemm_decode(x, w, out, mode)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
ops.gemm_decode(x, w, out, mode)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
