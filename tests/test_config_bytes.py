"""Dimensions, parameter counts and the decode byte model against SURVEY.md §8a/§8d."""
import pytest

from paper_2604_19877_b200 import APRIEL, PRESETS, TINY
from paper_2604_19877_b200 import roofline
from paper_2604_19877_b200.placement import FA, GDN, KDA, SWA, layer_kinds


def test_apriel_param_counts():
    assert APRIEL.mixer_params(FA) == pytest.approx(52.43e6, rel=1e-3)
    assert APRIEL.mixer_params(GDN) == pytest.approx(73.75e6, rel=1e-3)
    assert APRIEL.mixer_params(KDA) == pytest.approx(86.47e6, rel=1e-3)
    assert APRIEL.ffn_params() == pytest.approx(220.2e6, rel=1e-3)
    # the supernet (all four mixers per layer) is the paper's ~25B (R/PAPER.md:239)
    total = 48 * (2 * APRIEL.mixer_params(FA) + APRIEL.mixer_params(GDN) + APRIEL.mixer_params(KDA)
                  + APRIEL.ffn_params()) + 2 * APRIEL.vocab * APRIEL.hidden
    assert 24e9 < total < 26e9


def test_fused_widths():
    assert APRIEL.gdn_in_width == 10304 and APRIEL.gdn_conv_channels == 6144
    assert APRIEL.kda_in_width == 12576 and APRIEL.attn_qkv_width == 6144
    assert TINY.n_q_heads // TINY.n_kv_heads == APRIEL.n_q_heads // APRIEL.n_kv_heads == 4
    assert TINY.gdn_v_heads // TINY.gdn_k_heads == APRIEL.gdn_v_heads // APRIEL.gdn_k_heads == 4


def test_step_bytes_match_survey_table():
    kinds = layer_kinds(PRESETS["Reg|Lklhd-10"].layer_string)
    assert roofline.weight_bytes(APRIEL, kinds) / 1e9 == pytest.approx(29.26, abs=0.02)
    assert roofline.step_bytes(APRIEL, kinds, 64, 32768) / 1e9 == pytest.approx(50.4, abs=0.1)
    fa = layer_kinds(PRESETS["all-FA"].layer_string)
    assert roofline.weight_bytes(APRIEL, fa) / 1e9 == pytest.approx(27.52, abs=0.02)
    assert roofline.kv_token_bytes(APRIEL) == 4096


def test_kernel_launch_bytes():
    gd = roofline.kernel_launch_bytes(APRIEL, "gdn_decode", 64, 32768)
    assert gd == 64 * (2 * 32 * 128 * 128 * 4 + 2 * 6144 * 3 * 2 + (10304 + 4096) * 2)
    sw = roofline.kernel_launch_bytes(APRIEL, "swa_decode", 64, 32768)
    assert sw == 64 * (4096 * 4096 + 2 * 32 * 128 * 2)


def test_swiglu_interleave_roundtrip():
    """The fused gate/up weight layout (mode swiglu_il) and its prefill inverse are exact."""
    import torch
    from paper_2604_19877_b200 import ops
    N, K, h = 100, 8, 48
    w = torch.randn(2 * N, K)
    il = ops.interleave_swiglu(w, h)
    assert il.shape == (3 * 2 * h, K)
    x = torch.randn(5, K)
    assert torch.equal(ops.deinterleave_swiglu(x @ il.t(), N, h), x @ w.t())
    assert torch.equal(il.view(3, 2, h, K)[:, 0].reshape(-1, K)[:N], w[:N])
    assert not il.view(3, 2, h, K)[-1, :, N - 2 * h:].any()
