"""Pipeline wait breakdown of one decode-GEMM launch (producer empty-waits vs MMA full-waits)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_19877_b200 import _lib, ops  # noqa: E402

lib = _lib.load()
for spec in sys.argv[1:]:
    N, K, mode = spec.split(":")[0], spec.split(":")[1], (spec.split(":")[2] if spec.count(":") > 1 else "store")
    N, K = int(N), int(K)
    M = 64
    ws = [torch.randn(2 * N if mode == "swiglu" else N, K, device="cuda").to(torch.bfloat16) for _ in range(3)]
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    out = torch.zeros(8, M, N, device="cuda", dtype=torch.float32) if mode == "partial" else \
        torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    st = torch.zeros(148 * 8, dtype=torch.int64, device="cuda")
    for i in range(2):
        ops.gemm_decode(x, ws[i], out, mode)
    torch.cuda.synchronize()
    lib.sn_gemm_debug_stats(st.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ops.gemm_decode(x, ws[2], out, mode)
    e1.record()
    torch.cuda.synchronize()
    lib.sn_gemm_debug_stats(None)
    s = st.view(148, 8).double().cpu()
    act = s[:, 3] > 0
    s = s[act]
    t0 = s[:, 4:5]
    rel = torch.cat([s[:, 1:2], s[:, 5:]], 1)
    rel = (rel - t0) / 1.9e3  # clock64 cycles -> us at ~1.9 GHz, relative to the CTA's own entry
    print(f"  timeline us from CTA entry (min/mean/max): setup {rel[:,0].min():.2f}/{rel[:,0].mean():.2f}/{rel[:,0].max():.2f}"
          f"  first-stage {rel[:,1].min():.2f}/{rel[:,1].mean():.2f}/{rel[:,1].max():.2f}"
          f"  mma-done {rel[:,2].min():.2f}/{rel[:,2].mean():.2f}/{rel[:,2].max():.2f}"
          f"  exit {rel[:,3].min():.2f}/{rel[:,3].mean():.2f}/{rel[:,3].max():.2f}")
    print(f"{N}x{K} {mode}: {e0.elapsed_time(e1)*1e3:.1f} us event; CTAs {int(act.sum())}; "
          f"producer wait {s[:,0].mean()/1e3:.1f}k cyc; "
          f"MMA full-wait/total {s[:,2].mean()/1e3:.1f}k/{s[:,3].mean()/1e3:.1f}k cyc")
