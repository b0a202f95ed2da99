"""Time one decode GEMM shape under forced tilings (env SN_GEMM_FORCE="br,splits"), in a CUDA
graph over rotating weight copies (no L2 reuse), with the per-CTA pipeline counters."""
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "--one":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    from paper_2604_19877_b200 import _lib, ops
    N, K, mode = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    M = 64
    rows = 2 * N if mode.startswith("swiglu") else N
    nbuf = max(2, min(8, int(3e9 // (rows * K * 2))))
    Ws = [torch.randn(rows, K, device="cuda").to(torch.bfloat16) for _ in range(nbuf)]
    if mode == "swiglu_il":
        Ws = [ops.interleave_swiglu(w_, ops.gemm_swiglu_block(M, N, K)) for w_ in Ws]
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    out = torch.zeros(8, M, N, device="cuda") if mode == "partial" else torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    for i in range(3):
        ops.gemm_decode(x, Ws[i % nbuf], out, mode)
    it = 40
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        ops.gemm_decode(x, Ws[0], out, mode)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        for i in range(it):
            ops.gemm_decode(x, Ws[i % nbuf], out, mode)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / it * 1e3
    st = torch.zeros(148 * 8, dtype=torch.int64, device="cuda")
    _lib.load().sn_gemm_debug_stats(st.data_ptr())
    splits = ops.gemm_decode(x, Ws[1], out, mode)
    torch.cuda.synchronize()
    _lib.load().sn_gemm_debug_stats(None)
    c = st.view(148, 8).double().cpu()
    c = c[c[:, 4] > 0]
    print(f"  {N}x{K} {mode:9s} force={os.environ.get('SN_GEMM_FORCE', '-'):8s} cluster={os.environ.get('SN_GEMM_CLUSTER', '1')} "
          f"splits={splits}: {us:6.1f} us  {rows * K * 2 / us / 1e3:5.0f} GB/s  CTAs {len(c)}  "
          , flush=True)
    t = (c[:, [1, 5, 6, 7]] - c[:, 4:5]) / 1.9e3
    print("    us from entry (mean/max): producer-done %.1f/%.1f  first-stage %.1f/%.1f  mma-done %.1f/%.1f  epilogue-done %.1f/%.1f"
          % tuple(v for col in range(4) for v in (t[:, col].mean(), t[:, col].max())), flush=True)
else:
    for spec in sys.argv[1:]:
        N, K, mode, *forces = spec.split(":")
        print(f"{N}x{K} {mode}", flush=True)
        for f in [""] + forces:
            for cl in ("1",):
                env = dict(os.environ, SN_GEMM_CLUSTER=cl)
                if f:
                    env["SN_GEMM_FORCE"] = f
                subprocess.run([sys.executable, __file__, "--one", N, K, mode], env=env)
