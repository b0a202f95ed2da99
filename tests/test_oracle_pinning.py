"""Pin the CPU oracle before trusting it (the reference itself has no tests
or golden vectors for the mixer step, so the oracle is pinned against the third-party
realisation the paper's stack runs — FLA 0.5.1's own naive reference functions — and
against PyTorch SDPA for attention).  The FLA outputs are frozen in
tests/golden/fla_pinning.pt (tools/make_golden.py) so this also runs where FLA is absent."""
import math
import os

import pytest
import torch

from oracle.supernet_oracle import OracleSupernet, attention_ref, delta_rule_recurrent, rope
from paper_2604_19877_b200 import TINY
from paper_2604_19877_b200.placement import GDN, KDA, layer_kinds
from paper_2604_19877_b200.weights import init_weights

GOLD = os.path.join(os.path.dirname(__file__), "golden")
FLA = torch.load(os.path.join(GOLD, "fla_pinning.pt"))


def _max_rel(a, b):
    return ((a - b).abs().max() / b.abs().max()).item()


@pytest.mark.parametrize("variant", ["gdn", "kda"])
def test_recurrence_matches_fla_naive(variant):
    x = FLA["inputs"]
    g = x["g_scalar"] if variant == "gdn" else x["g_vec"]
    o, S = delta_rule_recurrent(x["q"], x["k"], x["v"], x["beta"], g, initial_state=x["h0"])
    ref = FLA[variant]
    assert _max_rel(o, ref["o"]) < 1e-5
    assert _max_rel(S, ref["S"]) < 1e-5
    # the chunked (WY / DPLR, C=64) forms FLA trains with agree with the same recurrence
    assert _max_rel(o, ref["o_chunk"]) < 1e-4
    assert _max_rel(S, ref["S_chunk"]) < 1e-4


def test_kda_with_broadcast_gate_is_gdn():
    x = FLA["inputs"]
    gs = x["g_scalar"]
    o1, S1 = delta_rule_recurrent(x["q"], x["k"], x["v"], x["beta"], gs, initial_state=x["h0"])
    o2, S2 = delta_rule_recurrent(x["q"], x["k"], x["v"], x["beta"], gs[..., None].expand_as(x["g_vec"]),
                                  initial_state=x["h0"])
    assert _max_rel(o1, o2) < 1e-6 and _max_rel(S1, S2) < 1e-6


@pytest.mark.parametrize("window", [0, 5])
def test_attention_matches_sdpa(window):
    g = torch.Generator().manual_seed(0)
    B, S, Hq, Hkv, D = 2, 11, 8, 2, 16
    q = torch.randn(B, Hq, D, generator=g)
    k = torch.randn(B, S, Hkv, D, generator=g)
    v = torch.randn(B, S, Hkv, D, generator=g)
    lo = S - window if window else 0
    ours = attention_ref(q, k[:, lo:], v[:, lo:], D ** -0.5)
    kk = k[:, lo:].transpose(1, 2).repeat_interleave(Hq // Hkv, 1)
    vv = v[:, lo:].transpose(1, 2).repeat_interleave(Hq // Hkv, 1)
    ref = torch.nn.functional.scaled_dot_product_attention(q[:, :, None], kk, vv)[:, :, 0]
    assert _max_rel(ours, ref) < 1e-5


def test_rope_is_rotate_half_and_norm_preserving():
    x = torch.randn(3, 2, 64)
    pos = torch.tensor([0, 7, 4096])
    inv = TINY.inv_freq().float()
    y = rope(x, pos, inv)
    assert torch.allclose(y[0], x[0])
    assert torch.allclose(y.norm(dim=-1), x.norm(dim=-1), rtol=1e-5)
    half = 32
    ang = 7 * inv[3]
    assert y[1, 0, 3].item() == pytest.approx((x[1, 0, 3] * math.cos(ang) - x[1, 0, 3 + half] * math.sin(ang)).item(),
                                              rel=1e-5)


@pytest.mark.parametrize("placement", ["AAAA", "ASKG"])
def test_oracle_reproduces_golden_tiny_logits(placement):
    """BASELINE.json configs 1/2: the oracle is deterministic and pinned to the committed fixture."""
    gold = torch.load(os.path.join(GOLD, "tiny_logits.pt"))
    kinds = layer_kinds(placement)
    o = OracleSupernet(TINY, kinds, init_weights(TINY, kinds, seed=0), batch=1, max_len=576)
    lg = o.run(gold["tokens"])
    g = gold[placement]
    assert torch.allclose(lg[0, g["positions"]], g["logits"], atol=1e-5, rtol=1e-5)
    for l, S in g["states"].items():
        assert torch.allclose(o.recurrent_state(l), S, atol=1e-5, rtol=1e-5)


def test_prefill_equals_stepwise():
    """The oracle's prefill is its decode loop: splitting a sequence gives identical logits."""
    kinds = layer_kinds("SGKA")
    w = init_weights(TINY, kinds, seed=3)
    toks = torch.randint(0, TINY.vocab, (2, 40), generator=torch.Generator().manual_seed(5))
    a = OracleSupernet(TINY, kinds, w, batch=2, max_len=40).run(toks)
    o = OracleSupernet(TINY, kinds, w, batch=2, max_len=40)
    b = torch.cat([o.run(toks[:, :17]), o.run(toks[:, 17:])], dim=1)
    assert torch.equal(a, b)


# ---------------------------------------------------------------- FLA module kernels
# tests/golden/fla_modules.pt holds the outputs of FLA 0.5.1's own gate functions, L2 norm,
# short causal conv (prefill + ShortConvolution.step) and FusedRMSNormGated, run on a B200 by
# tools/make_golden_fla_gpu.py (those FLA modules are Triton-only).  The oracle's restatements
# that gdn_core / kda_core call must reproduce them.
MOD = torch.load(os.path.join(GOLD, "fla_modules.pt"))


def test_gdn_gate_matches_fla():
    from oracle.supernet_oracle import gdn_gate
    x = MOD["gdn_gate"]
    ours = gdn_gate(x["a"], x["A_log"], x["dt_bias"])
    assert _max_rel(ours, x["naive"]) < 1e-6
    assert _max_rel(ours, x["fused"]) < 1e-5


def test_kda_gate_matches_fla():
    from oracle.supernet_oracle import kda_gate
    x = MOD["kda_gate"]
    ours = kda_gate(x["f"], x["A_log"], x["dt_bias"])
    assert _max_rel(ours, x["naive"]) < 1e-6
    assert _max_rel(ours, x["fused"]) < 1e-5


def test_l2norm_matches_fla():
    from oracle.supernet_oracle import l2norm
    x = MOD["l2norm"]
    assert _max_rel(l2norm(x["x"], x["eps"]), x["y"]) < 1e-5
    # the tiny row: eps inside the root, not a clamp on the norm
    assert torch.allclose(l2norm(x["x"][3], x["eps"]), x["y"][3], rtol=1e-4, atol=1e-6)


def test_short_conv_prefill_and_step_match_fla():
    """The oracle's conv step (history of the previous W-1 inputs, SiLU) run token by token
    reproduces FLA's prefill convolution, its final cache (the last W inputs) and three
    ShortConvolution.step calls from that cache."""
    from oracle.supernet_oracle import causal_conv_step
    x = MOD["short_conv"]
    w, xs = x["weight"], x["x"]
    B, T, C = xs.shape
    W = w.shape[1]
    hist = torch.zeros(B, C, W - 1)
    ys = []
    for t in range(T):
        y, hist = causal_conv_step(xs[:, t], hist, w)
        ys.append(y)
    assert _max_rel(torch.stack(ys, 1), x["y"]) < 1e-5
    assert torch.allclose(hist, x["cache_prefill"][..., 1:], atol=1e-6)
    for t in range(3):
        y, hist = causal_conv_step(x["steps"][t][:, 0], hist, w)
        assert _max_rel(y, x["y_steps"][t][:, 0]) < 1e-5
    assert torch.allclose(hist, x["cache_steps"][..., 1:], atol=1e-6)


@pytest.mark.parametrize("act", ["silu", "sigmoid"])
def test_gated_rmsnorm_matches_fla(act):
    from oracle.supernet_oracle import gated_rmsnorm
    x = MOD["gated_norm"]
    ours = gated_rmsnorm(x["o"], x["weight"], x["gate"], x["eps"], act)
    assert _max_rel(ours, x["swish" if act == "silu" else "sigmoid"]) < 1e-5
