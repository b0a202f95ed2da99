"""Supernet dimensions and the constants the paper leaves unstated.

Every constant the oracle and the kernels must agree on is pinned here once
(SURVEY.md App. A).  Sources:
  * Apriel-1.6 trunk: R/PAPER.md:175-182 (48 layers, d=5120, GQA 32q/8kv,
    d_h=128, SiLU FFN 14336, vocab 131072).
  * SWA window w=4096: R/PAPER.md:188-189, 1558-1563.
  * GDN 8 key heads / 32 value heads, d_k=d_v=128: R/PAPER.md:1595-1597
    (state kept per value head).
  * KDA 32 heads, d_h=128, low-rank gates d -> d_h -> n_h*d_h: R/PAPER.md:1610-1622.
  * Unstated, pinned from FLA 0.5.1 defaults: conv width 4, L2-norm eps 1e-6,
    gated-norm eps 1e-5, GDN out-gate silu / KDA sigmoid.
  * RoPE: rotate-half, theta 1e6 (not stated in the paper; App. A item 4).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, replace


@dataclass(frozen=True)
class SupernetConfig:
    name: str
    num_layers: int
    hidden: int
    vocab: int
    ffn: int
    # FA / SWA
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    window: int
    rope_theta: float
    # GDN
    gdn_k_heads: int
    gdn_v_heads: int
    gdn_head_dim: int
    # KDA
    kda_heads: int
    kda_head_dim: int
    kda_rank: int
    conv_width: int = 4
    norm_eps: float = 1e-5        # trunk RMSNorm
    mixer_norm_eps: float = 1e-5  # gated RMSNorm inside GDN/KDA
    l2_eps: float = 1e-6          # q/k L2 norm inside GDN/KDA
    page_size: int = 64           # KV page (tokens)
    chunk_size: int = 64          # chunked prefill chunk (C)

    # ---- derived widths of the fused projections (column layouts in include/sn_abi.h)
    @property
    def attn_qkv_width(self) -> int:
        return (self.n_q_heads + 2 * self.n_kv_heads) * self.head_dim

    @property
    def attn_o_in(self) -> int:
        return self.n_q_heads * self.head_dim

    @property
    def gdn_conv_channels(self) -> int:
        return (2 * self.gdn_k_heads + self.gdn_v_heads) * self.gdn_head_dim

    @property
    def gdn_in_width(self) -> int:  # [q | k | v | z | b | a]
        return 2 * self.gdn_k_heads * self.gdn_head_dim + 2 * self.gdn_v_heads * self.gdn_head_dim + 2 * self.gdn_v_heads

    @property
    def gdn_value_dim(self) -> int:
        return self.gdn_v_heads * self.gdn_head_dim

    @property
    def kda_dim(self) -> int:
        return self.kda_heads * self.kda_head_dim

    @property
    def kda_conv_channels(self) -> int:
        return 3 * self.kda_dim

    @property
    def kda_in_width(self) -> int:  # [q | k | v | f1 | g1 | b]
        return 3 * self.kda_dim + 2 * self.kda_rank + self.kda_heads

    def scaled(self, **kw) -> "SupernetConfig":
        return replace(self, **kw)

    # ---- parameter counts (per layer, per mixer) — cross-checked in tests against SURVEY.md §8a
    def mixer_params(self, kind: int) -> int:
        d = self.hidden
        if kind in (0, 1):
            return d * self.attn_qkv_width + self.attn_o_in * d
        if kind == 3:
            return (d * self.gdn_in_width + self.gdn_conv_channels * self.conv_width + 2 * self.gdn_v_heads
                    + self.gdn_head_dim + self.gdn_value_dim * d)
        if kind == 2:
            D, R, H = self.kda_head_dim, self.kda_rank, self.kda_heads
            return (d * self.kda_in_width + self.kda_conv_channels * self.conv_width + 2 * R * H * D + H * D
                    + H + H * D + D + self.kda_dim * d)
        raise ValueError(kind)

    def ffn_params(self) -> int:
        return 3 * self.hidden * self.ffn

    def inv_freq(self):
        import torch
        half = self.head_dim // 2
        return 1.0 / (self.rope_theta ** (torch.arange(0, half, dtype=torch.float64) * 2.0 / self.head_dim))


TINY = SupernetConfig(
    name="tiny",
    num_layers=4, hidden=256, vocab=4096, ffn=768,
    n_q_heads=4, n_kv_heads=1, head_dim=64, window=128, rope_theta=1e6,
    gdn_k_heads=1, gdn_v_heads=4, gdn_head_dim=64,
    kda_heads=4, kda_head_dim=64, kda_rank=64,
)

APRIEL = SupernetConfig(
    name="apriel-1.6-supernet",
    num_layers=48, hidden=5120, vocab=131072, ffn=14336,
    n_q_heads=32, n_kv_heads=8, head_dim=128, window=4096, rope_theta=1e6,
    gdn_k_heads=8, gdn_v_heads=32, gdn_head_dim=128,
    kda_heads=32, kda_head_dim=128, kda_rank=128,
)

CONFIGS = {"tiny": TINY, "apriel": APRIEL}


def attn_scale(cfg: SupernetConfig) -> float:
    return 1.0 / math.sqrt(cfg.head_dim)
