"""Algorithmic byte model of a decode step — the numerator of
every roofline fraction we report.

Per decode step of batch B at context T:
  weights: every GEMM weight read once in bf16 (selected mixer per layer, FFN,
           LM head; the embedding row gather is ignored);
  FA:      read (T+1) keys+values, i.e. 2*Hkv*D*2 B per token per layer, plus
           the appended token;
  SWA:     the same over min(T+1, w) ring slots;
  GDN/KDA: fp32 state read + write (2*Hv*D*D*4 B), conv tails read + write.
This is the ideal traffic; measured DRAM bytes above it are re-reads.
"""
from __future__ import annotations

from .config import SupernetConfig
from .placement import FA, GDN, KDA, SWA


def weight_bytes(cfg: SupernetConfig, kinds, elt: int = 2) -> int:
    n = sum(cfg.mixer_params(k) for k in kinds) + cfg.num_layers * cfg.ffn_params() + cfg.vocab * cfg.hidden
    return n * elt


def kv_token_bytes(cfg: SupernetConfig, elt: int = 2) -> int:
    return 2 * cfg.n_kv_heads * cfg.head_dim * elt


def mixer_state_bytes(cfg: SupernetConfig, kind: int, ctx: int, elt: int = 2) -> int:
    """Per sequence, per layer, per decode step."""
    if kind == FA:
        return (ctx + 1) * kv_token_bytes(cfg, elt)
    if kind == SWA:
        return (min(ctx, cfg.window) + 1) * kv_token_bytes(cfg, elt)
    W1 = cfg.conv_width - 1
    if kind == GDN:
        return 2 * cfg.gdn_v_heads * cfg.gdn_head_dim ** 2 * 4 + 2 * cfg.gdn_conv_channels * W1 * elt
    if kind == KDA:
        return 2 * cfg.kda_heads * cfg.kda_head_dim ** 2 * 4 + 2 * cfg.kda_conv_channels * W1 * elt
    raise ValueError(kind)


def step_bytes(cfg: SupernetConfig, kinds, B: int, ctx: int, elt: int = 2) -> int:
    return weight_bytes(cfg, kinds, elt) + B * sum(mixer_state_bytes(cfg, k, ctx, elt) for k in kinds)


def kernel_launch_bytes(cfg: SupernetConfig, name: str, B: int, ctx: int, elt: int = 2) -> int:
    """Algorithmic bytes of one launch of one of our mixer kernels (one layer, whole batch)."""
    if name == "gdn_decode":
        per = mixer_state_bytes(cfg, GDN, ctx, elt) + (cfg.gdn_in_width + cfg.gdn_value_dim) * elt
        return B * per
    if name == "kda_decode":
        per = mixer_state_bytes(cfg, KDA, ctx, elt) + (cfg.kda_in_width + cfg.kda_dim) * elt
        # second low-rank factors f2, g2 (+bias) read once per launch
        return B * per + (2 * cfg.kda_dim * cfg.kda_rank + cfg.kda_dim) * elt
    if name in ("fa_decode", "swa_decode"):
        keys = ctx + 1 if name == "fa_decode" else min(ctx + 1, cfg.window)
        return B * (keys * kv_token_bytes(cfg, elt) + 2 * cfg.n_q_heads * cfg.head_dim * elt)
    raise ValueError(name)


def role_step_bytes(cfg: SupernetConfig, kinds, role: str, B: int, ctx: int, elt: int = 2):
    """Algorithmic bytes per decode step of one kernel role of the step (the names the
    bench's KernelProbe records): mixer kernels as kernel_launch_bytes x layers of that kind;
    GEMM roles as weight bytes + bf16 activations in and out.  None for latency-bound glue
    (norms, RoPE/append, embed, argmax)."""
    d, F = cfg.hidden, cfg.ffn
    mixer = {"gdn_decode": [GDN], "kda_decode": [KDA], "fa_decode": [FA], "swa_decode": [SWA]}
    if role in mixer:
        n = sum(1 for k in kinds if k in mixer[role])
        return n * kernel_launch_bytes(cfg, role, B, ctx, elt)

    def gemm(N, K):
        return (N * K + B * (N + K)) * elt
    if role == "gemm_ffn_gate_up":
        return len(kinds) * gemm(2 * F, d)
    if role == "gemm_ffn_down":
        return len(kinds) * gemm(d, F)
    if role == "gemm_lm_head":
        return gemm(cfg.vocab, d)
    if role == "gemm_in_proj":
        width = {FA: cfg.attn_qkv_width, SWA: cfg.attn_qkv_width, GDN: cfg.gdn_in_width, KDA: cfg.kda_in_width}
        return sum(gemm(width[k], d) for k in kinds)
    if role == "gemm_out_proj":
        o_in = {FA: cfg.attn_o_in, SWA: cfg.attn_o_in, GDN: cfg.gdn_value_dim, KDA: cfg.kda_dim}
        return sum(gemm(d, o_in[k]) for k in kinds)
    if role == "chain":  # fused decode chains (csrc/sn_chain.cu): every projection of the step
        kda_gates = sum(1 for k in kinds if k == KDA) * 2 * gemm(cfg.kda_dim, cfg.kda_rank)
        return sum(role_step_bytes(cfg, kinds, r, B, ctx, elt) for r in
                   ("gemm_ffn_gate_up", "gemm_ffn_down", "gemm_lm_head", "gemm_in_proj", "gemm_out_proj")) + kda_gates
    return None
