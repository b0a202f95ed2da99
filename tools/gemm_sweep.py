"""Sweep split-K / batch for the decode GEMM inside CUDA graphs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_19877_b200 import ops  # noqa: E402


def timeit(fn, it=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=s):
        for _ in range(it):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it * 1e3


shapes = [(6144, 5120), (10304, 5120), (5120, 14336)]
if len(sys.argv) > 1:
    shapes = [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]]
for (N, K) in shapes:
    for M in (16, 64):
        nb = 4
        Ws = [torch.randn(N, K, device="cuda").to(torch.bfloat16) for _ in range(nb)]
        x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        out = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
        i = [0]
        def f():
            ops.gemm_decode(x, Ws[i[0] % nb], out, "store")
            i[0] += 1
        us = timeit(f)
        print(f"N={N} K={K} M={M}: {us:7.1f}us {N * K * 2 / us / 1e3:6.0f}GB/s", flush=True)
        del Ws
