"""Prefill attention kernel alone (Apriel heads: 32 q / 8 kv x 128): tokens/s and TFLOP/s of
the masked attention, causal (FA) and window 4096 (SWA), for one long sequence.
"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_19877_b200 import ops  # noqa: E402

Hq, Hkv, D = 32, 8, 128
for T in [int(x) for x in (sys.argv[1:] or ["4096", "16384"])]:
    q = torch.randn(T, Hq, D, device="cuda").to(torch.bfloat16)
    k = torch.randn(T, Hkv, D, device="cuda").to(torch.bfloat16)
    v = torch.randn(T, Hkv, D, device="cuda").to(torch.bfloat16)
    cu = torch.tensor([0, T], dtype=torch.int32, device="cuda")
    out = torch.empty(T, Hq * D, device="cuda", dtype=torch.bfloat16)
    for window in (0, 4096):
        ops.attn_prefill(q, k, v, cu, out, Hq, Hkv, D, window, 1 / math.sqrt(D))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            ops.attn_prefill(q, k, v, cu, out, Hq, Hkv, D, window, 1 / math.sqrt(D))
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        pairs = sum(min(i + 1, window) if window else i + 1 for i in range(T))
        flops = 4.0 * pairs * Hq * D
        print(f"tcgen05 T={T:6d} window={window:5d}: {ms:8.3f} ms  "
              f"{flops / ms / 1e9:7.1f} TFLOP/s")
