"""Deterministic random-init supernet weights (there are no checkpoints offline).

Every tensor is drawn from its own seeded generator keyed by (seed, layer,
mixer kind, tensor name), so layer l's FA weights are the same tensor whatever
placement is loaded — the supernet property (R/PAPER.md:239-241: every layer
holds weights for all four mixers; single-preset mode loads one of them,
R/PAPER.md:829-831).

Init (SURVEY.md §8d "Synthetic inputs"): Linear ~ N(0, 0.02^2); embedding
N(0, 1); RMSNorm weights 1 + N(0, 0.1^2) (non-trivial so the multiply is
exercised); causal conv taps U(-1/sqrt(W), 1/sqrt(W)) (nn.Conv1d default, not
DIL's identity, so every tap matters); GDN A_log = log U(1e-3, 16), KDA A_log =
log U(1, 16), dt_bias = softplus^-1(dt), dt ~ logU(1e-3, 1e-1) — the FLA
constructors (3P-FLA/layers/gated_deltanet.py, 3P-FLA/layers/kda.py __init__).
A_log and dt_bias are fp32; everything else is cast to the model dtype.

Fused layouts (documented column orders, include/sn_abi.h):
  attention qkv  [q Hq*D | k Hkv*D | v Hkv*D]
  GDN in-proj    [q Hk*D | k Hk*D | v Hv*D | z Hv*D | b Hv | a Hv]
  KDA in-proj    [q H*D | k H*D | v H*D | f1 R | g1 R | b H]
  FFN gate_up    [gate F | up F]
All matrices are nn.Linear-style [out, in].
"""
from __future__ import annotations

import math

import torch

from .config import SupernetConfig
from .placement import FA, GDN, KDA, SWA

_TENSOR_IDS = {
    "embed": 1, "final_norm": 2, "lm_head": 3, "norm1": 4, "norm2": 5, "ffn_gu": 6, "ffn_down": 7,
    "qkv": 10, "o": 11, "w_in": 12, "conv_w": 13, "A_log": 14, "dt_bias": 15, "norm_w": 16, "f2": 17,
    "g2": 18, "g2_b": 19,
}


def _seed(base: int, layer: int, kind: int, name: str) -> int:
    return (base * 1_000_003 + (layer + 1) * 10_007 + (kind + 1) * 101 + _TENSOR_IDS[name]) & 0x7FFF_FFFF


class _Draw:
    def __init__(self, base: int, device, dtype):
        self.base, self.device, self.dtype = base, torch.device(device), dtype

    def _gen(self, layer, kind, name):
        g = torch.Generator(device=self.device)
        g.manual_seed(_seed(self.base, layer, kind, name))
        return g

    def normal(self, shape, std, layer, kind, name, mean=0.0, dtype=None):
        g = self._gen(layer, kind, name)
        t = torch.randn(shape, generator=g, device=self.device, dtype=torch.float32)
        t = t.mul_(std).add_(mean)
        return t.to(dtype or self.dtype)

    def uniform(self, shape, lo, hi, layer, kind, name, dtype=None):
        g = self._gen(layer, kind, name)
        t = torch.rand(shape, generator=g, device=self.device, dtype=torch.float32)
        return (t * (hi - lo) + lo).to(dtype or self.dtype)


def _inv_softplus_dt(draw: _Draw, n, layer, kind):
    u = draw.uniform((n,), 0.0, 1.0, layer, kind, "dt_bias", dtype=torch.float32)
    dt = torch.exp(u * (math.log(0.1) - math.log(1e-3)) + math.log(1e-3)).clamp(min=1e-4)
    return dt + torch.log(-torch.expm1(-dt))


def init_trunk(cfg: SupernetConfig, seed: int = 0, device="cpu", dtype=torch.float32) -> dict:
    dr = _Draw(seed, device, dtype)
    d, V, F = cfg.hidden, cfg.vocab, cfg.ffn
    trunk = {
        "embed": dr.normal((V, d), 1.0, -1, -1, "embed"),
        "final_norm": dr.normal((d,), 0.1, -1, -1, "final_norm", mean=1.0),
        "lm_head": dr.normal((V, d), 0.02, -1, -1, "lm_head"),
        "layers": [],
    }
    for l in range(cfg.num_layers):
        trunk["layers"].append({
            "norm1": dr.normal((d,), 0.1, l, -1, "norm1", mean=1.0),
            "norm2": dr.normal((d,), 0.1, l, -1, "norm2", mean=1.0),
            "ffn_gu": dr.normal((2 * F, d), 0.02, l, -1, "ffn_gu"),
            "ffn_down": dr.normal((d, F), 0.02, l, -1, "ffn_down"),
        })
    return trunk


def init_mixer(cfg: SupernetConfig, layer: int, kind: int, seed: int = 0, device="cpu", dtype=torch.float32) -> dict:
    dr = _Draw(seed, device, dtype)
    d, W = cfg.hidden, cfg.conv_width
    cw = 1.0 / math.sqrt(W)
    if kind in (FA, SWA):
        return {
            "qkv": dr.normal((cfg.attn_qkv_width, d), 0.02, layer, kind, "qkv"),
            "o": dr.normal((d, cfg.attn_o_in), 0.02, layer, kind, "o"),
        }
    if kind == GDN:
        Hv, D = cfg.gdn_v_heads, cfg.gdn_head_dim
        return {
            "w_in": dr.normal((cfg.gdn_in_width, d), 0.02, layer, kind, "w_in"),
            "conv_w": dr.uniform((cfg.gdn_conv_channels, W), -cw, cw, layer, kind, "conv_w"),
            "A_log": torch.log(dr.uniform((Hv,), 1e-3, 16.0, layer, kind, "A_log", dtype=torch.float32)),
            "dt_bias": _inv_softplus_dt(dr, Hv, layer, kind),
            "norm_w": dr.normal((D,), 0.1, layer, kind, "norm_w", mean=1.0),
            "o": dr.normal((d, cfg.gdn_value_dim), 0.02, layer, kind, "o"),
        }
    if kind == KDA:
        H, D, R = cfg.kda_heads, cfg.kda_head_dim, cfg.kda_rank
        return {
            "w_in": dr.normal((cfg.kda_in_width, d), 0.02, layer, kind, "w_in"),
            "conv_w": dr.uniform((cfg.kda_conv_channels, W), -cw, cw, layer, kind, "conv_w"),
            "f2": dr.normal((H * D, R), 1.0 / math.sqrt(R), layer, kind, "f2"),
            "g2": dr.normal((H * D, R), 1.0 / math.sqrt(R), layer, kind, "g2"),
            "g2_b": dr.normal((H * D,), 0.02, layer, kind, "g2_b"),
            "A_log": torch.log(dr.uniform((H,), 1.0, 16.0, layer, kind, "A_log", dtype=torch.float32)),
            "dt_bias": _inv_softplus_dt(dr, H * D, layer, kind),
            "norm_w": dr.normal((D,), 0.1, layer, kind, "norm_w", mean=1.0),
            "o": dr.normal((d, cfg.kda_dim), 0.02, layer, kind, "o"),
        }
    raise ValueError(f"unknown mixer kind {kind}")


def init_weights(cfg: SupernetConfig, kinds, seed: int = 0, device="cpu", dtype=torch.float32) -> dict:
    """Trunk + the selected mixer of every layer (single-preset mode)."""
    w = init_trunk(cfg, seed, device, dtype)
    for l, k in enumerate(kinds):
        w["layers"][l]["mixer"] = init_mixer(cfg, l, k, seed, device, dtype)
    return w


def cast_weights(w, device=None, dtype=None):
    """Recursively move/cast; fp32 gate parameters (A_log, dt_bias) keep fp32."""
    if isinstance(w, dict):
        return {k: (v.to(device=device) if k in ("A_log", "dt_bias") and torch.is_tensor(v)
                    else cast_weights(v, device, dtype)) for k, v in w.items()}
    if isinstance(w, list):
        return [cast_weights(v, device, dtype) for v in w]
    if torch.is_tensor(w):
        return w.to(device=device, dtype=dtype if w.is_floating_point() else w.dtype)
    return w
