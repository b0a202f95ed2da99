"""CPU ORACLE for the Super Apriel per-layer mixer step — TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product: only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs may import it.  The product
path (paper_2604_19877_b200) has no CPU fallback and never imports this file.

What it restates.  The reference ships no implementation of the mixer step
(R/SPEC.md:8 scopes it out), so this is a definitional, token-by-token fp32
restatement of the paper's equations:
  * trunk (pre-norm residual, SiLU-gated FFN, final norm, LM head):
      R/PAPER.md:175-182, 855-856
  * FA: GQA softmax attention with RoPE, R/PAPER.md:1540-1556
  * SWA: same with the mask j in (t-w, t], R/PAPER.md:1558-1563 (App. A item 3)
  * GDN: S_t = e^{g_t}(I - b_t k k^T) S_{t-1} + b_t k v^T, fused QKVZ/BA
      projections, joint causal conv + SiLU, L2-normalised q/k, gated RMSNorm(z):
      R/PAPER.md:1565-1599
  * KDA: S_t = (I - b_t k k^T) diag(e^{g_t}) S_{t-1} + b_t k v^T, separate
      convs, low-rank per-channel gate and output gate: R/PAPER.md:1601-1625
Details the paper leaves open follow FLA 0.5.1 (third-party, not vendored by
the reference): gate formulas 3P-FLA/ops/gated_delta_rule/gate.py:20-45
and 3P-FLA/ops/kda/gate.py:26-54, recurrence 3P-FLA/ops/gated_delta_rule/naive.py:13-64
and 3P-FLA/ops/kda/naive.py:12-66, L2 norm 3P-FLA/modules/l2norm.py:40-43, conv step
3P-FLA/modules/conv/short_conv.py:201-243, gated norm 3P-FLA/modules/fused_norm_gate.py:94-100.

Parity pinning.  The reference has no tests or golden vectors for this path
("parity unpinned" by the reference itself).  This oracle is
pinned instead against FLA's own naive reference functions (recurrent and
chunked GDN/KDA, tests/test_oracle_pinning.py) and against PyTorch's
scaled_dot_product_attention for FA/SWA; the golden fixtures under
tests/golden/ are produced by tools/make_golden.py from this oracle.

Prefill here is simply T decode steps (the recurrent form is the definition);
the product's chunked/parallel prefill must agree with it.
"""
from __future__ import annotations

import math

import torch
import torch.nn.functional as F

FA, SWA, KDA, GDN = 0, 1, 2, 3


def rmsnorm(x, w, eps):
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * w


def l2norm(x, eps):
    return x * torch.rsqrt(x.pow(2).sum(-1, keepdim=True) + eps)


def rope(x, pos, inv_freq):
    """Rotate-half RoPE. x [B, H, D]; pos [B] int; inv_freq [D/2] fp32."""
    ang = pos.to(torch.float32)[:, None] * inv_freq[None, :]  # [B, D/2]
    cos, sin = torch.cos(ang)[:, None, :], torch.sin(ang)[:, None, :]
    half = x.shape[-1] // 2
    x1, x2 = x[..., :half], x[..., half:]
    return torch.cat([x1 * cos - x2 * sin, x2 * cos + x1 * sin], dim=-1)


def gdn_gate(a_raw, A_log, dt_bias):
    """GDN log-decay per value head: g = -exp(A_log) * softplus(a + dt_bias)
    (3P-FLA/ops/gated_delta_rule/gate.py:20-45, naive_gdn_gate).  a_raw [..., Hv]."""
    return -A_log.exp() * F.softplus(a_raw + dt_bias)


def kda_gate(f, A_log, dt_bias):
    """KDA log-decay per key channel: g = -exp(A_log[h]) * softplus(f + dt_bias[h, k])
    (3P-FLA/ops/kda/gate.py:26-54, naive_kda_gate).  f [..., H, K]; dt_bias [H*K]."""
    H = f.shape[-2]
    return -A_log.view(H, 1).exp() * F.softplus(f + dt_bias.view(H, -1))


def gated_rmsnorm(o, w, gate, eps, act):
    """Per-head RMSNorm(o) * w * act(gate), act 'silu' (GDN) or 'sigmoid' (KDA)
    (3P-FLA/modules/fused_norm_gate.py:94-100, FusedRMSNormGated)."""
    return rmsnorm(o, w, eps) * (F.silu(gate) if act == "silu" else torch.sigmoid(gate))


def causal_conv_step(x, hist, w):
    """One step of the SiLU causal conv.  x [B, C]; hist [B, C, W-1] (oldest first); w [C, W].
    Returns (y [B, C], new hist)."""
    window = torch.cat([hist, x[:, :, None]], dim=-1)  # [B, C, W]
    y = F.silu((window * w[None]).sum(-1))
    return y, window[:, :, 1:]


class OracleSupernet:
    """fp32 CPU oracle of the supernet for one fixed placement.

    weights: the structure produced by paper_2604_19877_b200.weights.init_weights
    (any float dtype; converted to fp32 here).  kinds: per-layer mixer kind.
    """

    def __init__(self, cfg, kinds, weights, batch: int, max_len: int, device="cpu"):
        """device: where the fp32 arithmetic runs.  "cpu" is the oracle proper; a CUDA device
        runs the SAME fp32 torch code (TF32 must be off — the Apriel-shaped parity tests assert
        it) only so that checks at Apriel widths finish in seconds.  Either way this is the
        checker, never the product."""
        self.cfg, self.kinds, self.B, self.max_len = cfg, tuple(kinds), batch, max_len
        self.device = torch.device(device)
        if self.device.type == "cuda" and torch.backends.cuda.matmul.allow_tf32:
            raise ValueError("oracle on CUDA needs torch.backends.cuda.matmul.allow_tf32 = False (fp32 checker)")
        f32 = lambda t: t.detach().to(self.device, torch.float32)
        self.w = _map_tensors(weights, f32)
        self.inv_freq = cfg.inv_freq().to(self.device, torch.float32)
        self.pos = 0
        # tensor-parallel emulation hook: applied to every row-parallel output (mixer out-proj,
        # FFN down) before the residual add; identity for the single-device oracle
        self.reduce = lambda t: t
        B, Hkv, D = batch, cfg.n_kv_heads, cfg.head_dim
        z = lambda *shape: torch.zeros(*shape, device=self.device)
        self.state = []
        for k in self.kinds:
            if k in (FA, SWA):
                self.state.append({"k": z(B, max_len, Hkv, D), "v": z(B, max_len, Hkv, D)})
            elif k == GDN:
                C, Hv, Dg = cfg.gdn_conv_channels, cfg.gdn_v_heads, cfg.gdn_head_dim
                self.state.append({"S": z(B, Hv, Dg, Dg), "hist": z(B, C, cfg.conv_width - 1)})
            else:
                C, H, Dk = cfg.kda_conv_channels, cfg.kda_heads, cfg.kda_head_dim
                self.state.append({"S": z(B, H, Dk, Dk), "hist": z(B, C, cfg.conv_width - 1)})

    # ------------------------------------------------------------ mixers
    def _attention(self, l, xn, kind):
        cfg, st, w = self.cfg, self.state[l], self.w["layers"][l]["mixer"]
        B, Hq, Hkv, D = xn.shape[0], cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim
        p = xn @ w["qkv"].T
        q = p[:, : Hq * D].view(B, Hq, D)
        k = p[:, Hq * D: (Hq + Hkv) * D].view(B, Hkv, D)
        v = p[:, (Hq + Hkv) * D:].view(B, Hkv, D)
        pos = torch.full((B,), self.pos, dtype=torch.long, device=self.device)
        q, k = rope(q, pos, self.inv_freq), rope(k, pos, self.inv_freq)
        st["k"][:, self.pos], st["v"][:, self.pos] = k, v
        lo = max(0, self.pos - cfg.window + 1) if kind == SWA else 0
        keys, vals = st["k"][:, lo: self.pos + 1], st["v"][:, lo: self.pos + 1]  # [B, S, Hkv, D]
        o = attention_ref(q, keys, vals, 1.0 / math.sqrt(D))
        return o.reshape(B, Hq * D) @ w["o"].T

    def _gdn(self, l, xn):
        st, w = self.state[l], self.w["layers"][l]["mixer"]
        o, st["hist"], st["S"] = gdn_core(self.cfg, xn @ w["w_in"].T, st["hist"], st["S"], w)
        return o @ w["o"].T

    def _kda(self, l, xn):
        st, w = self.state[l], self.w["layers"][l]["mixer"]
        o, st["hist"], st["S"] = kda_core(self.cfg, xn @ w["w_in"].T, st["hist"], st["S"], w)
        return o @ w["o"].T

    # ------------------------------------------------------------ step
    @torch.no_grad()
    def step(self, tokens):
        """One decode step for all B sequences (same position).  tokens [B] -> logits [B, V]."""
        cfg, w = self.cfg, self.w
        if self.pos >= self.max_len:
            raise ValueError("oracle max_len exceeded")
        x = w["embed"][torch.as_tensor(tokens, dtype=torch.long).to(self.device)]
        for l, kind in enumerate(self.kinds):
            lw = w["layers"][l]
            xn = rmsnorm(x, lw["norm1"], cfg.norm_eps)
            if kind in (FA, SWA):
                x = x + self.reduce(self._attention(l, xn, kind))
            elif kind == GDN:
                x = x + self.reduce(self._gdn(l, xn))
            else:
                x = x + self.reduce(self._kda(l, xn))
            xn = rmsnorm(x, lw["norm2"], cfg.norm_eps)
            gu = xn @ lw["ffn_gu"].T
            x = x + self.reduce((F.silu(gu[:, : cfg.ffn]) * gu[:, cfg.ffn:]) @ lw["ffn_down"].T)
        self.pos += 1
        return rmsnorm(x, w["final_norm"], cfg.norm_eps) @ w["lm_head"].T

    @torch.no_grad()
    def run(self, tokens):
        """tokens [B, T] -> logits [B, T, V] (teacher-forced, token by token)."""
        tokens = torch.as_tensor(tokens)
        return torch.stack([self.step(tokens[:, t]) for t in range(tokens.shape[1])], dim=1)

    def recurrent_state(self, layer):
        """[B, Hv, K, V] fp32 state of a GDN/KDA layer."""
        return self.state[layer]["S"]

    def conv_history(self, layer):
        return self.state[layer]["hist"]



def delta_step(S, q, k, v, beta, g):
    """One gated delta-rule step for all heads (the recurrence of R/PAPER.md:1575-1578 / 1606-1609).
    S [B, H, K, V]; q (already scaled), k [B, H, K]; v [B, H, V]; beta [B, H];
    g: log-decay, [B, H] (GDN, scalar per head) or [B, H, K] (KDA, per key channel).
    Returns (o [B, H, V], new S):  S <- diag(e^g) S;  S += k (beta (v - k^T S))^T;  o = S^T q."""
    decay = g.exp()[..., None] if g.dim() == 3 else g.exp()[:, :, None, None]
    S = S * decay
    u = beta[:, :, None] * (v - torch.einsum("bhk,bhkv->bhv", k, S))
    S = S + k[:, :, :, None] * u[:, :, None, :]
    return torch.einsum("bhk,bhkv->bhv", q, S), S


def delta_rule_recurrent(q, k, v, beta, g, initial_state=None, scale=None):
    """Token-by-token gated delta rule in FLA's calling convention (3P-FLA/ops/gated_delta_rule/
    naive.py:13-64 for g [B,T,H], 3P-FLA/ops/kda/naive.py:12-66 for g [B,T,H,K]):
    q,k [B,T,H,K], v [B,T,H,V], beta [B,T,H] -> (o [B,T,H,V], S [B,H,K,V]); q is scaled by K^-1/2."""
    B, T, H, K = q.shape
    scale = K ** -0.5 if scale is None else scale
    S = torch.zeros(B, H, K, v.shape[-1]) if initial_state is None else initial_state.float().clone()
    outs = []
    for t in range(T):
        o, S = delta_step(S, q[:, t].float() * scale, k[:, t].float(), v[:, t].float(), beta[:, t].float(),
                          g[:, t].float())
        outs.append(o)
    return torch.stack(outs, dim=1), S


def gdn_core(cfg, p, hist, S, w):
    """GDN mixer on the fused in-projection row(s) p [B, gdn_in_width] (R/PAPER.md:1565-1599).
    hist [B, C, W-1] conv history, S [B, Hv, K, V] state.  Returns (o [B, Hv*D] before the
    out-projection, new hist, new S)."""
    B, Hk, Hv, D = p.shape[0], cfg.gdn_k_heads, cfg.gdn_v_heads, cfg.gdn_head_dim
    C = cfg.gdn_conv_channels
    y, hist = causal_conv_step(p[:, :C], hist, w["conv_w"])
    q = y[:, : Hk * D].view(B, Hk, D)
    k = y[:, Hk * D: 2 * Hk * D].view(B, Hk, D)
    v = y[:, 2 * Hk * D:].view(B, Hv, D)
    z = p[:, C: C + Hv * D].view(B, Hv, D)
    b_raw = p[:, C + Hv * D: C + Hv * D + Hv]
    a_raw = p[:, C + Hv * D + Hv: C + Hv * D + 2 * Hv]
    G = Hv // Hk  # value head h reads key head h // G (GVA)
    q = (l2norm(q, cfg.l2_eps) / math.sqrt(D)).repeat_interleave(G, dim=1)
    k = l2norm(k, cfg.l2_eps).repeat_interleave(G, dim=1)
    g = gdn_gate(a_raw, w["A_log"], w["dt_bias"])  # [B, Hv]
    beta = torch.sigmoid(b_raw)
    o, S = delta_step(S, q, k, v, beta, g)
    o = gated_rmsnorm(o, w["norm_w"], z, cfg.mixer_norm_eps, "silu")
    return o.reshape(B, Hv * D), hist, S


def kda_core(cfg, p, hist, S, w):
    """KDA mixer on the fused in-projection row(s) p [B, kda_in_width] (R/PAPER.md:1601-1625)."""
    B, H, D, R = p.shape[0], cfg.kda_heads, cfg.kda_head_dim, cfg.kda_rank
    HD = H * D
    y, hist = causal_conv_step(p[:, : 3 * HD], hist, w["conv_w"])
    q, k, v = (y[:, i * HD: (i + 1) * HD].view(B, H, D) for i in range(3))
    f1 = p[:, 3 * HD: 3 * HD + R]
    g1 = p[:, 3 * HD + R: 3 * HD + 2 * R]
    b_raw = p[:, 3 * HD + 2 * R: 3 * HD + 2 * R + H]
    f = f1 @ w["f2"].T
    g = kda_gate(f.view(B, H, D), w["A_log"], w["dt_bias"])
    gate = (g1 @ w["g2"].T + w["g2_b"]).view(B, H, D)
    q = l2norm(q, cfg.l2_eps) / math.sqrt(D)
    k = l2norm(k, cfg.l2_eps)
    beta = torch.sigmoid(b_raw)
    o, S = delta_step(S, q, k, v, beta, g)
    o = gated_rmsnorm(o, w["norm_w"], gate, cfg.mixer_norm_eps, "sigmoid")
    return o.reshape(B, HD), hist, S


def attention_ref(q, keys, vals, scale):
    """softmax(q k^T * scale) v with GQA (query head h reads kv head h // G).
    q [B, Hq, D]; keys/vals [B, S, Hkv, D] (post-RoPE)."""
    B, Hq, D = q.shape
    Hkv = keys.shape[2]
    qg = q.view(B, Hkv, Hq // Hkv, D)
    sc = torch.einsum("bhgd,bshd->bhgs", qg, keys) * scale
    return torch.einsum("bhgs,bshd->bhgd", sc.softmax(-1), vals).reshape(B, Hq, D)


def _map_tensors(obj, fn):
    if isinstance(obj, dict):
        return {k: _map_tensors(v, fn) for k, v in obj.items()}
    if isinstance(obj, list):
        return [_map_tensors(v, fn) for v in obj]
    if torch.is_tensor(obj):
        return fn(obj)
    return obj
