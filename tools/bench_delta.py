"""GDN / KDA decode kernel in a CUDA graph at Apriel shapes (B=64), states rotating over
several layers so nothing is L2-resident: achieved GB/s vs the algorithmic bytes."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_19877_b200 import APRIEL, ops, roofline  # noqa: E402
from paper_2604_19877_b200.placement import GDN, KDA  # noqa: E402
from paper_2604_19877_b200.weights import init_mixer  # noqa: E402

cfg = APRIEL
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
L = 6
for kind in (GDN, KDA):
    w = {k: (v if k in ("A_log", "dt_bias") else v.to(torch.bfloat16)).cuda() for k, v in init_mixer(cfg, 0, kind).items()}
    Hv = cfg.gdn_v_heads if kind == GDN else cfg.kda_heads
    D = cfg.gdn_head_dim
    C = cfg.gdn_conv_channels if kind == GDN else cfg.kda_conv_channels
    N_in = cfg.gdn_in_width if kind == GDN else cfg.kda_in_width
    states = [torch.randn(B, Hv, D, D, device="cuda") * 0.05 for _ in range(L)]
    rings = [torch.randn(B, C, 4, device="cuda").to(torch.bfloat16) for _ in range(L)]
    proj = (torch.randn(B, N_in, device="cuda") * 0.5).to(torch.bfloat16)
    pos = torch.full((B,), 1000, dtype=torch.int32, device="cuda")
    out = torch.empty(B, Hv * D, device="cuda", dtype=torch.bfloat16)
    if kind == KDA:
        fgbuf = torch.empty(B, 2 * cfg.kda_dim, device="cuda", dtype=torch.bfloat16)

    def run(l):
        if kind == GDN:
            ops.gdn_decode(proj, rings[l], w["conv_w"], states[l], None, pos, w["A_log"], w["dt_bias"], w["norm_w"],
                           out, cfg.gdn_k_heads, Hv, D, 4, 1 / math.sqrt(D), 1e-6, 1e-5)
        else:  # the decode step's own gate-factor GEMMs, then the KDA kernel
            ops.kda_gate_factors(proj, w["f2"], w["g2"], fgbuf, Hv, D, cfg.kda_rank)
            ops.kda_decode(proj, fgbuf, rings[l], w["conv_w"], states[l], None, pos, w["A_log"], w["dt_bias"],
                           w["g2_b"], w["norm_w"], out, Hv, D, cfg.kda_rank, 4, 1 / math.sqrt(D), 1e-6, 1e-5)
    for l in range(L):
        run(l)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    reps = 4
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            for l in range(L):
                run(l)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (reps * L)
    name = "gdn_decode" if kind == GDN else "kda_decode"
    nbytes = roofline.kernel_launch_bytes(cfg, name, B, 32768)
    print(f"{name}: {us:7.1f} us/launch  {nbytes / us / 1e3:6.0f} GB/s  ({nbytes / 1e6:.0f} MB)")
