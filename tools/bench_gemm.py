"""Decode GEMM alone at the Apriel decode shapes: back-to-back launches inside one CUDA graph
(as in the decode step), distinct weight copies so nothing is an L2 hit; per-launch µs and
weight-stream GB/s for the built-in plan and forced (block rows, atoms per stage) variants.

  python tools/bench_gemm.py [M] [--variants]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_19877_b200 import APRIEL, ops  # noqa: E402
from paper_2604_19877_b200._lib import load  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 64
c = APRIEL
SHAPES = [("ffn_gate_up", c.ffn, c.hidden, "swiglu_il"), ("ffn_down", c.hidden, c.ffn, "partial"),
          ("gdn_in", c.gdn_in_width, c.hidden, "store"), ("gdn_out", c.hidden, c.gdn_value_dim, "partial"),
          ("kda_in", c.kda_in_width, c.hidden, "store"), ("attn_out", c.hidden, c.attn_o_in, "partial"),
          ("lm_head", c.vocab, c.hidden, "store")]


def time_gemm(N, K, mode, it=30):
    rows = -(-N // ops.gemm_swiglu_block(N)) * 2 * ops.gemm_swiglu_block(N) if mode == "swiglu_il" else N
    nbuf = max(2, min(8, int(3e9 // (rows * K * 2))))
    Ws = [torch.randn(rows, K, device="cuda").to(torch.bfloat16) for _ in range(nbuf)]
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    if mode == "partial":
        out = torch.zeros(8, M, N, device="cuda", dtype=torch.float32)
    else:
        out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if mode == "resid" else torch.bfloat16)
    for i in range(3):
        ops.gemm_decode(x, Ws[i % nbuf], out, mode)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=s):
        for i in range(it):
            ops.gemm_decode(x, Ws[i % nbuf], out, mode)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(3):
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / it)
    del Ws
    torch.cuda.empty_cache()
    return best * 1e3, rows * K * 2 / (best * 1e6)


lib = load()
variants = [(0, 0, 0)]
if "--variants" in sys.argv:
    variants += [(256, 1, 0), (256, 2, 0), (128, 1, 0), (128, 2, 0), (128, 4, 0), (64, 2, 0), (64, 4, 0), (64, 8, 0)]
if "--grid" in sys.argv:
    variants += [(0, 0, g) for g in (56, 64, 80, 96, 112, 120, 136, 148)]
if "--whole" in sys.argv:  # one whole block per CTA: grid = blocks
    variants += [(br, 0, -100) for br in (64, 80, 96, 112, 128, 144, 160, 192, 208, 224, 256)]
if "--dbg" in sys.argv:
    variants += [(0, 0, -1), (0, 0, -2), (0, 0, -3), (0, 0, -4)]
only = [a.split("=")[1] for a in sys.argv if a.startswith("--only=")]
for name, N, K, mode in SHAPES:
    if only and name not in only[0].split(","):
        continue
    for br, ks, grid in variants:
        if grid == -100:
            if mode == "swiglu_il":
                continue
            nb = -(-N // br)
            if nb > 148:
                continue
            grid = nb
        lib.sn_gemm_decode_tune(br, ks, 0, grid)
        plan = ops.gemm_decode_plan(M, N, K, mode)
        us, gbs = time_gemm(N, K, mode)
        print(f"{name:12s} N={N:6d} K={K:5d} {mode:9s} force=({br},{ks},{grid}) plan={plan} {us:7.1f} us {gbs:7.0f} GB/s",
              flush=True)
lib.sn_gemm_decode_tune(0, 0, 0, 0)
