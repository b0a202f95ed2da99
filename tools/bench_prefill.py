"""GDN prefill core (after prep): chunked WY on tensor cores vs the token-sequential scan,
Apriel head shapes, one sequence of T tokens, all 32 value heads."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_19877_b200 import ops  # noqa: E402

D, Hk, Hv = 128, 8, 32
for T in (512, 4096, 16384):
    qn = torch.nn.functional.normalize(torch.randn(T, Hk, D, device="cuda"), dim=-1) / math.sqrt(D)
    kn = torch.nn.functional.normalize(torch.randn(T, Hk, D, device="cuda"), dim=-1)
    qkv = torch.randn(T, (2 * Hk + Hv) * D, device="cuda").to(torch.bfloat16)
    glog = -torch.rand(T, Hv, device="cuda") * 0.3
    beta = torch.rand(T, Hv, device="cuda")
    cu = torch.tensor([0, T], dtype=torch.int32, device="cuda")
    S = torch.zeros(1, Hv, D, D, device="cuda")
    o = torch.empty(T, Hv, D, device="cuda")
    gexp = glog.exp()
    res = {}
    chunks, c0 = ops.chunk_plan([0, T])
    qb, kb = qn.to(torch.bfloat16), kn.to(torch.bfloat16)  # sn_delta_prep emits these in the model
    ws = None
    for name in ("chunk2", "scan"):
        def run():
            global ws
            if name == "chunk2":
                ws = ops.gdn_chunk_prefill2(qb, kb, qkv, 2 * Hk * D, glog, beta, chunks, c0, o, S, None, Hk, Hv, D,
                                            init_state=False, workspace=ws)
            else:
                ops.delta_scan(0, qn, kn, qkv, 2 * Hk * D, gexp, beta, o, S, None, cu, Hk, Hv, D, init_state=False)
        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            run()
        e1.record()
        torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) / 3
    flops = T / 64 * Hv * 2 * (64 * 64 * 128 * 2 + 64 * 128 * 64 + 64 * 64 * 64 + 64 * 128 * 64 * 3 + 64 * 64 * 64)
    print(f"GDN T={T:6d}: two-phase (tcgen05 chunk-local + state pass) {res['chunk2']:8.3f} ms "
          f"({flops / res['chunk2'] / 1e9:6.1f} TFLOP/s)   scan {res['scan']:8.3f} ms   "
          f"speed-up {res['scan'] / res['chunk2']:5.1f}x")

# KDA: per-channel gates, H = 32 heads of 128 (q/k per head), two-phase chunk vs scan
H = 32
for T in (512, 4096, 16384):
    qn = torch.nn.functional.normalize(torch.randn(T, H, D, device="cuda"), dim=-1) / math.sqrt(D)
    kn = torch.nn.functional.normalize(torch.randn(T, H, D, device="cuda"), dim=-1)
    qkv = torch.randn(T, 3 * H * D, device="cuda").to(torch.bfloat16)
    glog = -torch.rand(T, H, D, device="cuda") * 0.5
    beta = torch.rand(T, H, device="cuda")
    cu = torch.tensor([0, T], dtype=torch.int32, device="cuda")
    S = torch.zeros(1, H, D, D, device="cuda")
    o = torch.empty(T, H, D, device="cuda")
    gexp = glog.exp()
    chunks, c0 = ops.chunk_plan([0, T])
    qb, kb = qn.to(torch.bfloat16), kn.to(torch.bfloat16)  # sn_delta_prep emits these in the model
    ws = None
    res = {}
    for name in ("chunk2", "scan"):
        def run():
            global ws
            if name == "chunk2":
                ws = ops.kda_chunk_prefill2(qb, kb, qkv, 2 * H * D, glog, beta, chunks, c0, o, S, None, H, D,
                                            init_state=False, workspace=ws)
            else:
                ops.delta_scan(1, qn, kn, qkv, 2 * H * D, gexp, beta, o, S, None, cu, H, H, D, init_state=False)
        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            run()
        e1.record()
        torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) / 3
    print(f"KDA T={T:6d}: two-phase {res['chunk2']:8.3f} ms   scan {res['scan']:8.3f} ms   "
          f"speed-up {res['scan'] / res['chunk2']:5.1f}x")
