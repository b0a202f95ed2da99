"""Time one decode-GEMM shape (graph, back-to-back launches, rotating weights) under forced
plans (SN_GEMM_FORCE="rows,splits" is read per process, so each plan runs in a subprocess)."""
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "--one":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    from paper_2604_19877_b200 import ops
    N, K, mode = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    M = 64
    nbuf = 8
    Ws = [torch.randn(N, K, device="cuda").to(torch.bfloat16) for _ in range(nbuf)]
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    out = torch.zeros(8, M, N, device="cuda") if mode == "partial" else torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    for i in range(3):
        ops.gemm_decode(x, Ws[i % nbuf], out, mode)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=s):
        for i in range(40):
            ops.gemm_decode(x, Ws[i % nbuf], out, mode)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 40 * 1e3
    print(f"{os.environ.get('SN_GEMM_FORCE', 'auto'):>8s} N={N} K={K} {mode}: {us:7.1f} us  {N * K * 2 / us / 1e3:6.0f} GB/s")
    sys.exit(0)

N, K, mode = sys.argv[1], sys.argv[2], sys.argv[3]
for plan in ["auto"] + sys.argv[4:]:
    env = dict(os.environ)
    if plan != "auto":
        env["SN_GEMM_FORCE"] = plan
    subprocess.run([sys.executable, __file__, "--one", N, K, mode], env=env)
