"""Kernel-level parity at Apriel head shapes (D=128, GQA 32:8, GVA 8:32) — each
CUDA entry point against the oracle's math on the same inputs, plus the
bit-exact bookkeeping checks (KV slot placement, SWA ring, conv ring)."""
import math

import pytest
import torch

from oracle import bookkeeping as bk
from oracle.supernet_oracle import attention_ref, gdn_core, kda_core, rope
from paper_2604_19877_b200 import APRIEL, TINY
from paper_2604_19877_b200.placement import GDN, KDA

TOL = {torch.float32: 1e-4, torch.bfloat16: 2e-2}


def rel_err(a, b):
    a, b = a.detach().float().cpu(), b.detach().float().cpu()
    return ((a - b).abs().max() / b.abs().max().clamp_min(1e-6)).item()


def _ops():
    from paper_2604_19877_b200 import ops
    return ops


def _rand_pool(B, max_blocks, Hkv, P, D, dtype, gen, extra_pages=7):
    """Random K/V pool with a shuffled (non-contiguous) block table."""
    n_pages = B * max_blocks + extra_pages
    perm = torch.randperm(n_pages, generator=gen)[: B * max_blocks].to(torch.int32).view(B, max_blocks)
    k = torch.randn(n_pages, Hkv, P, D, generator=gen).to(dtype)
    v = torch.randn(n_pages, Hkv, P, D, generator=gen).to(dtype)
    return perm, k, v


def _gather_keys(pool, bt_row, n_keys, P):
    """[n_keys, Hkv, D] of logical slots 0..n_keys-1."""
    idx = torch.arange(n_keys)
    return pool[bt_row[idx // P].long(), :, idx % P]


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("window", [0, 4096])
@pytest.mark.parametrize("lens", [[1, 63, 64, 65], [1000, 4113, 31, 2048], [8191, 129, 4096, 5000]])
def test_attn_decode_apriel(dtype, window, lens):
    ops = _ops()
    gen = torch.Generator().manual_seed(7)
    B, Hq, Hkv, D, P = len(lens), 32, 8, 128, 64
    max_len = max(lens)
    max_blocks = math.ceil((window if window else max_len) / P)
    bt, kp, vp = _rand_pool(B, max_blocks, Hkv, P, D, dtype, gen)
    q = torch.randn(B, Hq, D, generator=gen).to(dtype)
    seq = torch.tensor(lens, dtype=torch.int32)
    scale = 1 / math.sqrt(D)
    ref = []
    for b in range(B):
        n = min(lens[b], window) if window else lens[b]
        keys = _gather_keys(kp.float(), bt[b], n, P)[None]
        vals = _gather_keys(vp.float(), bt[b], n, P)[None]
        ref.append(attention_ref(q[b:b + 1].float(), keys, vals, scale))
    ref = torch.cat(ref)
    from paper_2604_19877_b200.model import choose_split
    for split_pages in (1, 4, 16):
        max_splits = math.ceil(max_blocks / split_pages)
        ws = torch.empty(ops.attn_decode_workspace_bytes(B, Hq, Hkv, D, max_splits) // 4, device="cuda")
        ctr = torch.zeros(B * Hkv, dtype=torch.int32, device="cuda")
        out = torch.empty(B, Hq * D, dtype=dtype, device="cuda")
        ops.attn_decode(q.cuda(), kp.cuda(), vp.cuda(), bt.cuda(), seq.cuda(), out, ws, ctr, Hq, Hkv, D, P, window,
                        split_pages, max_splits, scale)
        torch.cuda.synchronize()
        err = rel_err(out.view(B, Hq, D), ref)
        assert err <= TOL[dtype], (split_pages, err)
        assert int(ctr.abs().sum()) == 0, "split counters must be re-armed to zero"


@pytest.mark.gpu
@pytest.mark.parametrize("window", [0, 128])
def test_rope_kv_append_slots_bit_exact(window):
    """Every row lands in exactly the (page, offset) the bookkeeping oracle names; SWA rows older
    than the window are not written; q/k rotation matches the oracle RoPE."""
    ops = _ops()
    cfg = TINY
    gen = torch.Generator().manual_seed(3)
    B, T, Hq, Hkv, D, P = 2, 300, cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim, cfg.page_size
    max_blocks = (window // P) if window else math.ceil(T / P)
    n_pages = B * max_blocks + 3
    bt = torch.randperm(n_pages, generator=gen)[: B * max_blocks].to(torch.int32).view(B, max_blocks)
    qkv = torch.randn(B * T, (Hq + 2 * Hkv) * D, generator=gen)
    row_seq = torch.arange(B, dtype=torch.int32).repeat_interleave(T)
    row_pos = torch.arange(T, dtype=torch.int32).repeat(B)
    seq_lens = torch.full((B,), T, dtype=torch.int32)
    inv = cfg.inv_freq().float()
    sentinel = -7.0
    kc = torch.full((n_pages, Hkv, P, D), sentinel, device="cuda")
    vc = torch.full_like(kc, sentinel)
    q_out = torch.empty(B * T, Hq, D, device="cuda")
    k_out = torch.empty(B * T, Hkv, D, device="cuda")
    v_out = torch.empty(B * T, Hkv, D, device="cuda")
    ops.rope_kv_append(qkv.cuda(), row_seq.cuda(), row_pos.cuda(), seq_lens.cuda(), inv.cuda(), q_out, k_out, v_out,
                       kc, vc, bt.cuda(), Hq, Hkv, D, P, window)
    torch.cuda.synchronize()
    kc, vc, k_out, v_out = kc.cpu(), vc.cpu(), k_out.cpu(), v_out.cpu()
    written = torch.zeros(n_pages, P, dtype=torch.bool)
    for b in range(B):
        for p in range(T):
            r = b * T + p
            if window and p < T - window:
                continue
            page, off = bk.swa_slot(bt[b].tolist(), p, window, P) if window else bk.fa_slot(bt[b].tolist(), p, P)
            assert torch.equal(kc[page, :, off], k_out[r]), (b, p)
            assert torch.equal(vc[page, :, off], v_out[r]), (b, p)
            written[page, off] = True
    assert torch.all(kc[~written[:, None, :, None].expand_as(kc)] == sentinel)
    # RoPE values vs oracle
    pos = row_pos.long()
    k_ref = rope(qkv[:, Hq * D:(Hq + Hkv) * D].view(-1, Hkv, D), pos, inv)
    q_ref = rope(qkv[:, :Hq * D].view(-1, Hq, D), pos, inv)
    assert rel_err(k_out, k_ref) <= 1e-5 and rel_err(q_out.cpu(), q_ref) <= 1e-5
    if window:
        ring = bk.swa_ring_contents(T, window)
        for s, p in enumerate(ring):
            page, off = bt[0, s // P].item(), s % P
            assert torch.equal(kc[page, :, off], k_out[p])


def _delta_weights(cfg, kind, gen, dtype):
    from paper_2604_19877_b200.weights import init_mixer
    w = init_mixer(cfg, 0, kind, seed=int(torch.randint(0, 1000, (1,), generator=gen)))
    return {k: (v if k in ("A_log", "dt_bias") else v.to(dtype)) for k, v in w.items()}


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("kind", [GDN, KDA])
@pytest.mark.parametrize("B", [3, 64])
@pytest.mark.parametrize("cfg", [APRIEL, TINY], ids=["apriel", "tiny"])
def test_delta_decode_steps(cfg, kind, B, dtype):
    """Several decode steps of the fused GDN/KDA kernel vs oracle gdn_core/kda_core, from a random
    non-zero state and conv history (including positions < W-1 where the ring must read zeros)."""
    ops = _ops()
    gen = torch.Generator().manual_seed(11 + kind)
    if B == 64 and cfg is not APRIEL:
        pytest.skip("B=64 (both delta-rule CTA widths) at Apriel shapes only")
    w = _delta_weights(cfg, kind, gen, dtype)
    if kind == GDN:
        Hv, D, C, width = cfg.gdn_v_heads, cfg.gdn_head_dim, cfg.gdn_conv_channels, cfg.gdn_in_width
    else:
        Hv, D, C, width = cfg.kda_heads, cfg.kda_head_dim, cfg.kda_conv_channels, cfg.kda_in_width
    W = cfg.conv_width
    S0 = torch.randn(B, Hv, D, D, generator=gen) * 0.1
    wf = {k: v.float() for k, v in w.items()}
    S_ref, hist = S0.clone(), torch.zeros(B, C, W - 1)
    S_dev = S0.transpose(-1, -2).contiguous().cuda()   # device layout [B, Hv, V, K]
    ring = torch.zeros(B, C, W, dtype=dtype, device="cuda")
    positions = torch.zeros(B, dtype=torch.int32, device="cuda")
    out = torch.empty(B, Hv * D, dtype=dtype, device="cuda")
    wd = {k: v.cuda() for k, v in w.items()}
    for step in range(6):
        p = (torch.randn(B, width, generator=gen) * 0.5).to(dtype)
        positions.fill_(step)
        if kind == GDN:
            o_ref, hist, S_ref = gdn_core(cfg, p.float(), hist, S_ref, wf)
            ops.gdn_decode(p.cuda(), ring, wd["conv_w"], S_dev, None, positions, wd["A_log"], wd["dt_bias"],
                           wd["norm_w"], out, cfg.gdn_k_heads, Hv, D, W, 1 / math.sqrt(D), cfg.l2_eps,
                           cfg.mixer_norm_eps)
        else:
            o_ref, hist, S_ref = kda_core(cfg, p.float(), hist, S_ref, wf)
            pc = torch.zeros(B, -(-width // 8) * 8, dtype=dtype, device="cuda")[:, :width]  # 16-byte row pitch
            pc.copy_(p)
            fg = torch.empty(B, 2 * Hv * D, dtype=dtype, device="cuda")
            ops.kda_gate_factors(pc, wd["f2"], wd["g2"], fg, Hv, D, cfg.kda_rank)
            ops.kda_decode(pc, fg, ring, wd["conv_w"], S_dev, None, positions, wd["A_log"], wd["dt_bias"],
                           wd["g2_b"], wd["norm_w"], out, Hv, D, cfg.kda_rank, W, 1 / math.sqrt(D), cfg.l2_eps,
                           cfg.mixer_norm_eps)
        torch.cuda.synchronize()
        assert rel_err(out, o_ref) <= TOL[dtype], (step, rel_err(out, o_ref))
        assert rel_err(S_dev.transpose(-1, -2), S_ref) <= TOL[dtype]
    # conv ring holds exactly the last W-1 inputs at slot pos % W (bit-exact, they are copies)
    ring_c = ring.cpu()
    for d in range(1, W):
        pos = 6 - d
        assert torch.equal(ring_c[:, :, bk.conv_ring_slot(pos, W)].float(), hist[:, :, W - 1 - d])


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("rows,vocab", [(1, 4096), (3, 16392), (64, 131072), (5, 100000)])
def test_argmax_matches_torch_first_occurrence(dtype, rows, vocab):
    """sn_argmax (a cluster of CTAs per row for large vocabularies) against torch.argmax: the
    first occurrence on ties, including ties across the CTAs of a row; -1 for idle slots; an
    all-NaN row gives token 0."""
    from paper_2604_19877_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(rows * vocab)
    x = torch.randn(rows, vocab, device="cuda", generator=g).to(dtype)
    if rows >= 3:  # ties: the max value at several positions spread over the row
        for r in range(rows):
            m = x[r].float().max().item() + 1.0
            for j in (vocab - 1, vocab // 2 + 5, 7 + r):
                x[r, j] = m
    out = torch.empty(rows, dtype=torch.int32, device="cuda")
    ops.argmax(x, out)
    assert torch.equal(out.long(), torch.argmax(x.float(), dim=-1))
    pos = torch.arange(rows, dtype=torch.int32, device="cuda")
    pos[0] = -1  # idle slot
    ops.argmax(x, out, pos)
    assert out[0].item() == -1 and torch.equal(out[1:].long(), torch.argmax(x[1:].float(), dim=-1))
    x[0] = float("nan")
    ops.argmax(x, out)
    assert out[0].item() == 0
