"""Head-parallel sharding with the real kernels on one GPU: every rank's slice of a mixer
(dist.shard_mixer, local head counts from dist.tp_config) runs through the CUDA decode
kernels, and the sum of the ranks' out-projection partials equals the unsharded mixer —
the decomposition the NCCL all-reduce after the out-projection relies on."""
import math

import pytest
import torch

from paper_2604_19877_b200 import APRIEL
from paper_2604_19877_b200.dist import shard_mixer, tp_config
from paper_2604_19877_b200.placement import GDN, KDA
from paper_2604_19877_b200.weights import init_mixer


def _run_delta(cfg, kind, w, x, S0):
    from paper_2604_19877_b200 import ops
    B = x.shape[0]
    dev = "cuda"
    wd = {k: v.to(dev) for k, v in w.items()}
    proj = x @ wd["w_in"].t()
    if kind == GDN:
        Hk, Hv, D, C = cfg.gdn_k_heads, cfg.gdn_v_heads, cfg.gdn_head_dim, cfg.gdn_conv_channels
    else:
        Hk = Hv = cfg.kda_heads
        D, C = cfg.kda_head_dim, cfg.kda_conv_channels
    ring = torch.zeros(B, C, cfg.conv_width, device=dev, dtype=x.dtype)
    S = S0.clone()
    pos = torch.zeros(B, dtype=torch.int32, device=dev)
    out = torch.empty(B, Hv * D, device=dev, dtype=x.dtype)
    if kind == GDN:
        ops.gdn_decode(proj, ring, wd["conv_w"], S, None, pos, wd["A_log"], wd["dt_bias"], wd["norm_w"], out, Hk, Hv,
                       D, cfg.conv_width, 1 / math.sqrt(D), cfg.l2_eps, cfg.mixer_norm_eps)
    else:
        fg = torch.empty(B, 2 * Hv * D, dtype=x.dtype, device=dev)
        ops.kda_gate_factors(proj, wd["f2"], wd["g2"], fg, Hv, D, cfg.kda_rank)
        ops.kda_decode(proj, fg, ring, wd["conv_w"], S, None, pos, wd["A_log"], wd["dt_bias"], wd["g2_b"],
                       wd["norm_w"], out, Hv, D, cfg.kda_rank, cfg.conv_width, 1 / math.sqrt(D), cfg.l2_eps,
                       cfg.mixer_norm_eps)
    return (out.float() @ wd["o"].float().t()), S


@pytest.mark.gpu
@pytest.mark.parametrize("kind", [GDN, KDA])
@pytest.mark.parametrize("world", [2, 8])
def test_delta_mixer_head_parallel(kind, world):
    cfg = APRIEL
    torch.manual_seed(0)
    # fp32 I/O: the sharded and unsharded in-projections then produce the same per-column values
    # (bf16 rounding would differ between GEMM shapes and blur the comparison)
    w = init_mixer(cfg, 0, kind)
    B = 4
    x = (torch.randn(B, cfg.hidden) * 0.5).cuda()
    H = cfg.gdn_v_heads if kind == GDN else cfg.kda_heads
    D = cfg.gdn_head_dim if kind == GDN else cfg.kda_head_dim
    S0 = (torch.randn(B, H, D, D) * 0.05).cuda()
    full, S_full = _run_delta(cfg, kind, w, x, S0)
    local = tp_config(cfg, world)
    h = H // world
    acc = torch.zeros_like(full)
    for r in range(world):
        part, S_r = _run_delta(local, kind, shard_mixer(cfg, kind, w, world, r), x,
                               S0[:, r * h:(r + 1) * h].contiguous())
        acc += part
        ref_s = S_full[:, r * h:(r + 1) * h]
        assert ((S_r - ref_s).abs().max() / ref_s.abs().max()).item() < 1e-4
    torch.cuda.synchronize()
    assert ((acc - full).abs().max() / full.abs().max()).item() < 1e-4
