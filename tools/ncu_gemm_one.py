"""One decode-GEMM shape launched a few times (for ncu -k dgemm --launch-skip 2 -c 1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_19877_b200 import ops  # noqa: E402

N, K, mode, M = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 64
rows = -(-N // ops.gemm_swiglu_block(N)) * 2 * ops.gemm_swiglu_block(N) if mode == "swiglu_il" else N
Ws = [torch.randn(rows, K, device="cuda").to(torch.bfloat16) for _ in range(3)]
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if mode == "resid" else torch.bfloat16)
ws = ops.gemm_decode_workspace(M, "cuda")
for i in range(4):
    ops.gemm_decode(x, Ws[i % 3], out, mode, ws)
torch.cuda.synchronize()
