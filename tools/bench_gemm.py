"""Decode GEMM: tcgen05 kernel vs cuBLAS (torch.mm) at the Apriel decode shapes, B=64."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_19877_b200 import ops

M = int(sys.argv[1]) if len(sys.argv) > 1 else 64
shapes = [("ffn_gu(swiglu_il)", 14336, 5120, "swiglu_il"), ("ffn_gu(swiglu)", 14336, 5120, "swiglu"), ("ffn_gu(partial)", 28672, 5120, "partial"),
          ("ffn_down(partial)", 5120, 14336, "partial"),
          ("gdn_in(partial)", 10304, 5120, "partial"), ("gdn_out(partial)", 5120, 4096, "partial"),
          ("attn_qkv(partial)", 6144, 5120, "partial"), ("kda_in(partial)", 12576, 5120, "partial"),
          ("lm_head", 131072, 5120, "store")]
for name, N, K, mode in shapes:
    rows = 2 * N if mode.startswith("swiglu") else N
    nbuf = max(2, min(8, int(3e9 // (rows * K * 2))))
    Ws = [torch.randn(rows, K, device="cuda").to(torch.bfloat16) for _ in range(nbuf)]
    if mode == "swiglu_il":
        Ws = [ops.interleave_swiglu(w_, ops.gemm_swiglu_block(M, N, K)) for w_ in Ws]
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    if mode == "partial":
        out = torch.zeros(8, M, N, device="cuda", dtype=torch.float32)
    else:
        out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if mode == "resid" else torch.bfloat16)
    res = {}
    splits = ops.gemm_decode_splits(M, N, K, mode) if mode == "partial" else 1
    for impl in ("sn", "cublas"):
        def run(i):
            if impl == "sn":
                ops.gemm_decode(x, Ws[i % nbuf], out, mode)
            else:
                y = x @ Ws[i % nbuf].t()
        for i in range(5):
            run(i)
        torch.cuda.synchronize()
        it = 40
        graph = torch.cuda.CUDAGraph()  # time inside a graph: no host launch overhead (as in the decode step)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            run(0)
        torch.cuda.synchronize()
        with torch.cuda.graph(graph, stream=s):
            for i in range(it):
                run(i)
        graph.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        graph.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / it * 1e3
        res[impl] = (us, rows * K * 2 / us / 1e3)
    print(f"{name:18s} N={N:6d} K={K:5d} splits={splits}  "
          f"sn {res['sn'][0]:7.1f}us {res['sn'][1]:6.0f}GB/s   cublas {res['cublas'][0]:7.1f}us {res['cublas'][1]:6.0f}GB/s")
    del Ws
