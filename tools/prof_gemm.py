"""One-shot decode GEMM launches for ncu (profile window = cudaProfilerStart/Stop)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_19877_b200 import ops
M = 64
cases = [("gdn_in", 10304, 5120, "store"), ("attn_qkv", 6144, 5120, "store"), ("ffn_down", 5120, 14336, "resid")]
bufs = []
for name, N, K, mode in cases:
    w = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if mode == "resid" else torch.bfloat16)
    bufs.append((w, x, out, mode))
    ops.gemm_decode(x, w, out, mode)
    y = x @ w.t()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for w, x, out, mode in bufs:
    ops.gemm_decode(x, w, out, mode)
    y = x @ w.t()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
