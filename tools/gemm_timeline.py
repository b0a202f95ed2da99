"""Per-CTA timeline of one decode-GEMM launch (sn_gemm_debug_stats clock64 counters):
CTA entry, producer done, last MMA issued, epilogue done — relative to each CTA's own
entry, in microseconds at ~1.9 GHz.  python tools/gemm_timeline.py N K mode [force]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_19877_b200 import _lib, ops  # noqa: E402

N, K, mode = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
lib = _lib.load()
M = 64
ws = [torch.randn(N, K, device="cuda").to(torch.bfloat16) for _ in range(4)]
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
out = torch.zeros(8, M, N, device="cuda") if mode == "partial" else torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
for i in range(3):
    ops.gemm_decode(x, ws[i], out, mode)
torch.cuda.synchronize()
st = torch.zeros(148 * 8, dtype=torch.int64, device="cuda")
lib.sn_gemm_debug_stats(st.data_ptr())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
ops.gemm_decode(x, ws[3], out, mode)
e1.record()
torch.cuda.synchronize()
lib.sn_gemm_debug_stats(None)
s = st.view(148, 8).double().cpu()
act = s[:, 4] > 0
s = s[act]
clk = torch.cuda.clock_rate() * 1e-3 if hasattr(torch.cuda, "clock_rate") else 1.9  # GHz
clk = 1.9
rel = lambda c: ((s[:, c] - s[:, 4]) / (clk * 1e3))  # per-CTA clock (SM clocks are not synchronised)
print(f"{N}x{K} {mode}: {e0.elapsed_time(e1) * 1e3:.1f} us (event), {int(act.sum())} CTAs")
for name, c in (("producer done", 1), ("last MMA", 6), ("epilogue done", 7)):
    r = rel(c)
    print(f"  {name:14s} min {r.min():6.2f}  mean {r.mean():6.2f}  max {r.max():6.2f} us")
