"""Same-box per-kernel comparison against the paper stack's sm100 kernels installed in the image
(the paper serves with vLLM + FlashInfer; FlashInfer 0.6.11 ships a GDN decode
kernel and the trtllm-gen paged decode attention).  Library code, used here only as the
comparison arm; nothing of it is on our path.

  * GDN decode, Apriel shapes (8 key / 32 value heads x 128, fp32 state [B, HV, V, K] — the
    layout both use): flashinfer.gated_delta_rule_decode_pretranspose (the delta-rule core with
    q/k L2 norm and gates) vs our sn_gdn_decode, which also runs the causal conv update and the
    gated RMSNorm.  Algorithmic bytes: the state read + write dominate both.
  * Paged decode attention, 32 q / 8 kv heads x 128, bf16 HND pages of 64 tokens:
    flashinfer.trtllm_batch_decode_with_kv_cache vs our sn_attn_decode, at B=64 x 4096 keys
    (the SWA layers' read volume) and B=23 x 32K (all-FA at capacity).

CUDA graphs of several launches over rotating buffers (nothing L2-resident), events.
Prints one line per case; a case whose library kernel is unavailable offline says so.
"""
import math
import os
import sys
import traceback

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_19877_b200 import APRIEL, ops, roofline  # noqa: E402
from paper_2604_19877_b200.weights import init_mixer  # noqa: E402
from paper_2604_19877_b200.placement import GDN  # noqa: E402


def graph_us(fn, n_inner, reps=5):
    fn(0)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=s):
        for i in range(n_inner):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / n_inner)
    return best


def gdn_case(B=64, L=6):
    import flashinfer
    cfg = APRIEL
    Hk, Hv, D = cfg.gdn_k_heads, cfg.gdn_v_heads, cfg.gdn_head_dim
    w = {k: (v if k in ("A_log", "dt_bias") else v.to(torch.bfloat16)).cuda() for k, v in init_mixer(cfg, 0, GDN).items()}
    states = [torch.randn(B, Hv, D, D, device="cuda") * 0.05 for _ in range(L)]
    rings = [torch.randn(B, cfg.gdn_conv_channels, 4, device="cuda").to(torch.bfloat16) for _ in range(L)]
    proj = (torch.randn(B, cfg.gdn_in_width, device="cuda") * 0.5).to(torch.bfloat16)
    pos = torch.full((B,), 1000, dtype=torch.int32, device="cuda")
    out = torch.empty(B, Hv * D, device="cuda", dtype=torch.bfloat16)
    ours = graph_us(lambda i: ops.gdn_decode(proj, rings[i % L], w["conv_w"], states[i % L], None, pos, w["A_log"],
                                             w["dt_bias"], w["norm_w"], out, Hk, Hv, D, 4, 1 / math.sqrt(D), 1e-6,
                                             1e-5), 4 * L)
    q = torch.randn(B, 1, Hk, D, device="cuda").to(torch.bfloat16)
    k = torch.randn(B, 1, Hk, D, device="cuda").to(torch.bfloat16)
    v = torch.randn(B, 1, Hv, D, device="cuda").to(torch.bfloat16)
    a = torch.randn(B, 1, Hv, device="cuda").to(torch.bfloat16)
    b = torch.randn(B, 1, Hv, device="cuda").to(torch.bfloat16)
    o = torch.empty(B, 1, Hv, D, device="cuda", dtype=torch.bfloat16)
    from flashinfer.gdn_decode import gated_delta_rule_decode_pretranspose as fi_gdn
    fi = graph_us(lambda i: fi_gdn(
        q, k, v, states[i % L], w["A_log"], a, w["dt_bias"].float(), b, scale=1 / math.sqrt(D), output=o,
        use_qk_l2norm=True), 4 * L)
    nbytes = roofline.kernel_launch_bytes(cfg, "gdn_decode", B, 32768)
    print(f"GDN decode B={B}: ours {ours:6.1f} us ({nbytes / ours / 1e3:5.0f} GB/s, conv + norm included) | "
          f"flashinfer gated_delta_rule_decode_pretranspose {fi:6.1f} us ({nbytes / fi / 1e3:5.0f} GB/s) | "
          f"ratio {fi / ours:.2f}x")


def attn_case(B, keys, L=4):
    import flashinfer
    cfg = APRIEL
    Hq, Hkv, D, P = cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim, cfg.page_size
    nb = -(-keys // P)
    kc = [torch.randn(B * nb, Hkv, P, D, device="cuda").to(torch.bfloat16) for _ in range(L)]
    vc = [torch.randn(B * nb, Hkv, P, D, device="cuda").to(torch.bfloat16) for _ in range(L)]
    bt = torch.arange(B * nb, dtype=torch.int32, device="cuda").view(B, nb)
    lens = torch.full((B,), keys, dtype=torch.int32, device="cuda")
    q = torch.randn(B, Hq, D, device="cuda").to(torch.bfloat16)
    out = torch.empty(B, Hq * D, device="cuda", dtype=torch.bfloat16)
    from paper_2604_19877_b200.model import choose_split
    sp, ms = choose_split(nb, B * Hkv)
    ws = torch.empty(ops.attn_decode_workspace_bytes(B, Hq, Hkv, D, ms) // 4 + 1, device="cuda")
    ctr = torch.zeros(B * Hkv, dtype=torch.int32, device="cuda")
    ours = graph_us(lambda i: ops.attn_decode(q, kc[i % L], vc[i % L], bt, lens, out, ws, ctr, Hq, Hkv, D, P, 0, sp, ms,
                                              1 / math.sqrt(D)), 2 * L)
    fws = torch.zeros(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    fo = torch.empty(B, Hq, D, device="cuda", dtype=torch.bfloat16)
    from flashinfer.decode import trtllm_batch_decode_with_kv_cache as fi_attn
    fi = graph_us(lambda i: fi_attn(
        q, (kc[i % L], vc[i % L]), fws, bt, lens, keys, bmm1_scale=1 / math.sqrt(D), out=fo, kv_layout="HND"), 2 * L)
    nbytes = B * (keys * 4096 + 2 * Hq * D * 2)
    print(f"paged decode attention B={B} x {keys} keys: ours {ours:7.1f} us ({nbytes / ours / 1e3:5.0f} GB/s) | "
          f"flashinfer trtllm_batch_decode_with_kv_cache {fi:7.1f} us ({nbytes / fi / 1e3:5.0f} GB/s) | "
          f"ratio {fi / ours:.2f}x")


if __name__ == "__main__":
    for name, fn in (("gdn", lambda: gdn_case()), ("attn 64x4096", lambda: attn_case(64, 4096)),
                     ("attn 23x32K", lambda: attn_case(23, 32768))):
        try:
            fn()
        except Exception as e:  # the library kernel may need artifacts that cannot be fetched offline
            print(f"{name}: flashinfer comparison unavailable: {type(e).__name__}: {str(e).splitlines()[0][:200]}")
            traceback.print_exc(limit=2, file=sys.stderr)
        torch.cuda.empty_cache()
