"""Decode GEMM (sn_gemm_decode: tcgen05 for bf16, CUDA-core tiles for fp32) vs a float64 torch
reference on the same operands: every epilogue (store, residual add, K-split fp32 slabs summed
by the norm, fused SwiGLU, fused RoPE + KV append), ragged N, batch 1..128, determinism, graph
replay."""
import math

import pytest
import torch

from oracle import bookkeeping as bk
from oracle.supernet_oracle import rope
from paper_2604_19877_b200 import APRIEL, TINY, ops

TOL = {torch.bfloat16: 8e-3, torch.float32: 1e-5}


def _ref(x, w):
    return x.double() @ w.double().t()


def rel(a, b):
    return ((a.double() - b.double()).abs().max() / b.double().abs().max().clamp_min(1e-6)).item()


def _operands(M, N, K, dtype, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(M, K, device="cuda", generator=g).to(dtype)
    w = (torch.randn(N, K, device="cuda", generator=g) * 0.05).to(dtype)
    return x, w


@pytest.mark.gpu
@pytest.mark.parametrize("M", [1, 7, 16, 33, 64, 100, 128])
@pytest.mark.parametrize("N,K", [(300, 256), (5120, 4096), (1000, 1024), (131072, 512), (10304, 5120),
                                 (6144, 5120), (5120, 14336)])
def test_gemm_store(M, N, K):
    x, w = _operands(M, N, K, torch.bfloat16, M * 7 + N)
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ops.gemm_decode(x, w, out, "store")
    torch.cuda.synchronize()
    assert rel(out, _ref(x, w)) < TOL[torch.bfloat16]


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("M", [1, 64, 128])
@pytest.mark.parametrize("F,K", [(768, 512), (14336, 5120), (1000, 256)])
def test_gemm_swiglu_il(dtype, M, F, K):
    x, w = _operands(M, 2 * F, K, dtype, 3)
    out = torch.empty(M, F, device="cuda", dtype=dtype)
    wk = ops.interleave_swiglu(w, ops.gemm_swiglu_block(F))
    ops.gemm_decode(x, wk, out, "swiglu_il")
    torch.cuda.synchronize()
    gu = _ref(x, w)
    ref = torch.nn.functional.silu(gu[:, :F]) * gu[:, F:]
    assert rel(out, ref) < TOL[dtype]


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("M", [3, 64])
@pytest.mark.parametrize("N,K", [(640, 4096), (5120, 14336), (304, 64), (5120, 4096)])
def test_gemm_resid_partial_deterministic(dtype, M, N, K):
    """"resid" adds into the residual in place; "partial" writes S K-split slabs that
    sn_add_rmsnorm sums in slab order — both deterministic, both equal to x @ w.T."""
    x, w = _operands(M, N, K, dtype, 5)
    r0 = torch.randn(M, N, device="cuda")
    outs = []
    for _ in range(2):
        r = r0.clone()
        ops.gemm_decode(x, w, r, "resid")
        outs.append(r)
    slabs = torch.empty(8, M, N, device="cuda")
    S = ops.gemm_decode(x, w, slabs, "partial")
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1]), "the GEMM must be deterministic"
    tol = 5e-5 if dtype == torch.float32 else 5e-4
    ref = _ref(x, w)
    assert rel(outs[0] - r0, ref) < tol
    assert 1 <= S <= 8 and S == ops.gemm_decode_plan(M, N, K, "partial")["splits"] or dtype == torch.float32
    assert rel(slabs[:S].sum(0), ref) < tol
    nw = torch.rand(N, device="cuda").to(dtype) + 0.5
    out = torch.empty(M, N, device="cuda", dtype=dtype)
    resid = r0.clone()
    ops.add_rmsnorm(None, resid, nw, out, 1e-5, partials=slabs, nsplit=S)
    torch.cuda.synchronize()
    ref_resid = r0.double() + slabs[:S].double().sum(0)
    assert (resid.double() - ref_resid).abs().max().item() < 1e-4
    ref_out = ref_resid * torch.rsqrt(ref_resid.pow(2).mean(-1, keepdim=True) + 1e-5) * nw.double()
    assert rel(out, ref_out) < (1e-2 if dtype == torch.bfloat16 else 1e-5)


@pytest.mark.gpu
def test_gemm_graph_replay_bit_identical():
    """Captured and replayed many times: same bits each time, counters stay zero."""
    M, N, K = 64, 10304, 5120
    x, w = _operands(M, N, K, torch.bfloat16, 17)
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ops.gemm_decode(x, w, out, "store")
    first = out.clone()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=s):
        ops.gemm_decode(x, w, out, "store")
    for _ in range(5):
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, first)


@pytest.mark.gpu
def test_gemm_plans_balance_the_sms():
    """Every Apriel decode projection keeps most SMs streaming (>= 100 of 148 CTAs busy)."""
    cfg = APRIEL
    for N, K, mode in ((cfg.gdn_in_width, cfg.hidden, "store"), (cfg.hidden, cfg.gdn_value_dim, "partial"),
                       (cfg.ffn, cfg.hidden, "swiglu_il"), (cfg.hidden, cfg.ffn, "partial"),
                       (cfg.vocab, cfg.hidden, "store"), (cfg.attn_qkv_width, cfg.hidden, "attn_in"),
                       (cfg.kda_in_width, cfg.hidden, "store")):
        p = ops.gemm_decode_plan(64, N, K, mode)
        assert p["grid"] >= 96 and p["blocks"] * p["splits"] >= p["grid"], (N, K, p)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("cfg,window", [(APRIEL, 0), (APRIEL, 4096), (TINY, 0), (TINY, 128)])
@pytest.mark.parametrize("M", [1, 5, 64])
def test_gemm_attn_in_rope_kv_append(dtype, cfg, window, M):
    """Fused attention in-projection: q == RoPE(x Wq^T), and k / v land bit-exactly in the
    (page, offset) of the bookkeeping oracle; a position past the block table is not written and
    raises the error flag."""
    Hq, Hkv, D, P = cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim, cfg.page_size
    K = cfg.hidden
    N = (Hq + 2 * Hkv) * D
    x, w0 = _operands(M, N, K, dtype, 23)
    w = ops.rope_pair_interleave(w0, Hq, Hkv, D)
    gen = torch.Generator().manual_seed(4)
    max_len = 9000
    max_blocks = window // P if window else math.ceil(max_len / P)
    n_pages = M * max_blocks + 5
    bt = torch.randperm(n_pages, generator=gen)[: M * max_blocks].to(torch.int32).view(M, max_blocks)
    pos = torch.randint(0, max_len, (M,), generator=gen, dtype=torch.int32)
    if M > 1:
        pos[1] = max_blocks * P if not window else pos[1]  # past the table (FA): skipped + flagged
    sentinel = -3.0
    kc = torch.full((n_pages, Hkv, P, D), sentinel, device="cuda", dtype=dtype)
    vc = torch.full_like(kc, sentinel)
    q = torch.empty(M, Hq, D, device="cuda", dtype=dtype)
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    inv = cfg.inv_freq().float()
    ops.gemm_decode_attn_in(x, w, pos.cuda(), inv.cuda(), q, kc, vc, bt.cuda(), Hq, Hkv, D, P, window, err)
    torch.cuda.synchronize()
    ref = _ref(x, w0).float().cpu()
    pl = pos.long()
    q_ref = rope(ref[:, :Hq * D].view(M, Hq, D), pl, inv)
    k_ref = rope(ref[:, Hq * D:(Hq + Hkv) * D].view(M, Hkv, D), pl, inv)
    v_ref = ref[:, (Hq + Hkv) * D:].view(M, Hkv, D)
    assert rel(q.cpu(), q_ref) < TOL[dtype] * 2
    kc, vc = kc.cpu(), vc.cpu()
    written = torch.zeros(n_pages, P, dtype=torch.bool)
    for m in range(M):
        p = int(pos[m])
        if not window and p >= max_blocks * P:
            continue
        page, off = bk.swa_slot(bt[m].tolist(), p, window, P) if window else bk.fa_slot(bt[m].tolist(), p, P)
        assert rel(kc[page, :, off], k_ref[m]) < TOL[dtype] * 2
        assert rel(vc[page, :, off], v_ref[m]) < TOL[dtype] * 2
        written[page, off] = True
    assert torch.all(kc[~written[:, None, :, None].expand_as(kc)] == sentinel)
    assert int(err.item()) == (1 if (M > 1 and not window) else 0)
