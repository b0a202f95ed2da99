"""Tensor-core prefill attention (sn_attn_prefill, bf16) vs an fp32 reference of the same
masked softmax attention: packed ragged sequences (tiles straddling sequence boundaries),
causal (FA) and sliding-window (SWA, keys i-w < j <= i) masks, GQA 4:1, D = 64 / 128."""
import math

import pytest
import torch

TOL = 2e-2


def reference(q, k, v, lens, window, scale):
    Hq, Hkv = q.shape[1], k.shape[1]
    G = Hq // Hkv
    out, t0 = [], 0
    for L in lens:
        qs, ks, vs = (x[t0:t0 + L].float().transpose(0, 1) for x in (q, k, v))  # [H, L, D]
        ks, vs = ks.repeat_interleave(G, 0), vs.repeat_interleave(G, 0)
        s = qs @ ks.transpose(1, 2) * scale
        i = torch.arange(L)[:, None]
        j = torch.arange(L)[None, :]
        ok = j <= i
        if window > 0:
            ok &= j > i - window
        s = s.masked_fill(~ok, float("-inf"))
        out.append((s.softmax(-1) @ vs).transpose(0, 1))
        t0 += L
    return torch.cat(out, 0)


@pytest.mark.gpu
@pytest.mark.parametrize("D", [128, 64])
@pytest.mark.parametrize("window", [0, 100])
@pytest.mark.parametrize("lens", [[1], [64], [130], [37, 200, 5, 64, 91], [700]])
def test_attn_prefill_tc(D, window, lens):
    from paper_2604_19877_b200 import ops
    Hq, Hkv = 8, 2
    g = torch.Generator().manual_seed(sum(lens) + D + window)
    T = sum(lens)
    q = torch.randn(T, Hq, D, generator=g).to(torch.bfloat16)
    k = torch.randn(T, Hkv, D, generator=g).to(torch.bfloat16)
    v = torch.randn(T, Hkv, D, generator=g).to(torch.bfloat16)
    cu = torch.tensor([0] + list(torch.tensor(lens).cumsum(0)), dtype=torch.int32)
    scale = 1.0 / math.sqrt(D)
    out = torch.empty(T, Hq * D, dtype=torch.bfloat16, device="cuda")
    ops.attn_prefill(q.cuda(), k.cuda(), v.cuda(), cu.cuda(), out, Hq, Hkv, D, window, scale)
    torch.cuda.synchronize()
    ref = reference(q, k, v, lens, window, scale).reshape(T, Hq * D)
    err = ((out.float().cpu() - ref).abs().max() / ref.abs().max()).item()
    assert err < TOL, err


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("D", [128, 64])
@pytest.mark.parametrize("window", [0, 100])
def test_attn_prefill_continuation(dtype, D, window):
    """New tokens appended to live sequences: keys are each sequence's cached prefix (from the
    first position the window can still see) plus the new tokens, packed by cu_k; the result
    must equal rows P.. of a one-shot prefill of the whole sequence."""
    from paper_2604_19877_b200 import ops
    Hq, Hkv = 8, 2
    prefix, new = [0, 150, 37], [70, 20, 130]
    g = torch.Generator().manual_seed(D + window)
    scale = 1.0 / math.sqrt(D)
    qs, ks, vs, ref_rows, cu_q, cu_k, q_off = [], [], [], [], [0], [0], []
    for P, N in zip(prefix, new):
        q = torch.randn(P + N, Hq, D, generator=g).to(dtype)
        k = torch.randn(P + N, Hkv, D, generator=g).to(dtype)
        v = torch.randn(P + N, Hkv, D, generator=g).to(dtype)
        ref_rows.append(reference(q, k, v, [P + N], window, scale)[P:])
        k0 = max(0, P - window) if window else 0
        qs.append(q[P:])
        ks.append(k[k0:])
        vs.append(v[k0:])
        cu_q.append(cu_q[-1] + N)
        cu_k.append(cu_k[-1] + P + N - k0)
        q_off.append(P - k0)
    q, k, v = torch.cat(qs), torch.cat(ks), torch.cat(vs)
    out = torch.empty(q.shape[0], Hq * D, dtype=dtype, device="cuda")
    i32 = dict(dtype=torch.int32, device="cuda")
    ops.attn_prefill(q.cuda(), k.cuda(), v.cuda(), torch.tensor(cu_q, **i32), out, Hq, Hkv, D, window, scale,
                     cu_k=torch.tensor(cu_k, **i32), q_off=torch.tensor(q_off, **i32))
    torch.cuda.synchronize()
    ref = torch.cat(ref_rows).reshape(q.shape[0], Hq * D)
    err = ((out.float().cpu() - ref).abs().max() / ref.abs().max()).item()
    assert err < (TOL if dtype == torch.bfloat16 else 1e-4), err


@pytest.mark.gpu
@pytest.mark.parametrize("window", [0, 300])
def test_attn_prefill_rising_scores(window):
    """Key norms growing along the sequence: the running row max keeps moving by more than
    the lazy-rescale headroom (2^8), so O is rescaled many times (and sometimes not)."""
    from paper_2604_19877_b200 import ops
    Hq, Hkv, D, T = 8, 2, 128, 1100
    g = torch.Generator().manual_seed(7 + window)
    ramp = torch.linspace(0.1, 8.0, T)[:, None, None]
    q = torch.randn(T, Hq, D, generator=g).to(torch.bfloat16)
    k = (torch.randn(T, Hkv, D, generator=g) * ramp).to(torch.bfloat16)
    v = torch.randn(T, Hkv, D, generator=g).to(torch.bfloat16)
    cu = torch.tensor([0, T], dtype=torch.int32)
    scale = 1.0 / math.sqrt(D)
    out = torch.empty(T, Hq * D, dtype=torch.bfloat16, device="cuda")
    ops.attn_prefill(q.cuda(), k.cuda(), v.cuda(), cu.cuda(), out, Hq, Hkv, D, window, scale)
    torch.cuda.synchronize()
    ref = reference(q, k, v, [T], window, scale).reshape(T, Hq * D)
    err = ((out.float().cpu() - ref).abs().max() / ref.abs().max()).item()
    assert err < TOL, err
