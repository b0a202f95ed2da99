"""Torch-facing wrappers over the C ABI (include/sn_abi.h).

Each wrapper checks shapes/dtypes/devices, then passes raw device pointers and
the current CUDA stream.  Nothing here computes on the CPU: a tensor that is
not on a CUDA device is an error.
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib
from ._lib import (SN_BF16, SN_CHAIN_GEMM, SN_CHAIN_NORM, SN_F32, ChainPhase, SN_GEMM_ATTN_IN, SN_GEMM_PARTIAL, SN_GEMM_RESID, SN_GEMM_STORE, SN_GEMM_SWIGLU_IL,
                   call)

_DT = {torch.bfloat16: SN_BF16, torch.float32: SN_F32}


def dtype_code(dt: torch.dtype) -> int:
    try:
        return _DT[dt]
    except KeyError:
        raise TypeError(f"unsupported I/O dtype {dt}; use bfloat16 or float32") from None


def _p(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("libsn100 ops need CUDA tensors (no CPU fallback)")
    return t.data_ptr()


def _s():
    return torch.cuda.current_stream().cuda_stream


def embed(tokens, table, residual, seq_lens=None, positions=None, inv_freq=None, rope_cs=None):
    """residual = table[tokens]; with seq_lens / positions the decode-step prologue; rope_cs
    ([rows, D/2, 2] fp32) also receives the step's rotary (cos, sin) table."""
    assert tokens.dtype == torch.int32 and residual.dtype == torch.float32
    half = rope_cs.shape[1] if rope_cs is not None else 0
    call("sn_embed", _p(tokens), _p(table), _p(residual), _p(seq_lens), _p(positions), _p(inv_freq), _p(rope_cs),
         half, tokens.numel(), table.shape[1], dtype_code(table.dtype), _s())


def add_rmsnorm(delta, residual, weight, out, eps, partials=None, nsplit=0):
    """residual += delta + sum(partials[:nsplit]) (slab order); out = rmsnorm(residual) * weight."""
    rows, dim = residual.shape
    if nsplit:
        assert partials is not None and partials.dtype == torch.float32 and partials.numel() >= nsplit * rows * dim
    call("sn_add_rmsnorm", _p(delta), _p(partials) if nsplit else None, int(nsplit), _p(residual), _p(weight),
         _p(out), rows, dim, eps, dtype_code(out.dtype), _s())


def argmax(logits, out_tokens, positions=None):
    """out_tokens = argmax over the vocabulary; -1 for idle slots (positions < 0)."""
    rows, vocab = logits.shape
    call("sn_argmax", _p(logits), rows, vocab, _p(out_tokens), _p(positions), dtype_code(logits.dtype), _s())


def rope_kv_append(qkv, row_seq, row_pos, seq_lens, inv_freq, q_out, k_out, v_out, k_cache, v_cache, block_table,
                   Hq, Hkv, D, page_size, window, pair_il=False):
    """qkv: [rows, (Hq+2Hkv)D] (dtype of the cache); pair_il: q / k columns in the rotary-pair
    interleaved order of the decode in-projection weights (rope_pair_interleave)."""
    rows = q_out.shape[0]
    call("sn_rope_kv_append", _p(qkv), _p(row_seq), _p(row_pos), _p(seq_lens), _p(inv_freq), _p(q_out), _p(k_out),
         _p(v_out), _p(k_cache), _p(v_cache), _p(block_table), rows, Hq, Hkv, D, page_size, block_table.shape[1],
         window, int(pair_il), dtype_code(q_out.dtype), _s())


def attn_decode_workspace_bytes(B, Hq, Hkv, D, max_splits):
    return _lib.load().sn_attn_decode_workspace_bytes(B, Hq, Hkv, D, max_splits)


def attn_decode(q, k_cache, v_cache, block_table, seq_lens, out, workspace, counters, Hq, Hkv, D, page_size, window,
                split_pages, max_splits, scale):
    B = seq_lens.shape[0]
    code = dtype_code(q.dtype)
    call("sn_attn_decode", _p(q), _p(k_cache), _p(v_cache), _p(block_table), _p(seq_lens), _p(out), _p(workspace),
         _p(counters), B, Hq, Hkv, D, page_size, block_table.shape[1], window, split_pages, max_splits, scale, code,
         _s())


def attn_prefill(q, k, v, cu_seqlens, out, Hq, Hkv, D, window, scale, cu_k=None, q_off=None):
    """Packed prefill attention; with cu_k / q_off the keys are a separate per-sequence packing
    (continuation: cached prefix + new tokens), see include/sn_abi.h."""
    call("sn_attn_prefill", _p(q), _p(k), _p(v), _p(cu_seqlens), _p(cu_k), _p(q_off), _p(out),
         cu_seqlens.numel() - 1, q.shape[0], k.shape[0], Hq, Hkv, D, window, scale, dtype_code(q.dtype), _s())


def gdn_decode(proj, conv_ring, conv_w, state, slot_idx, positions, A_log, dt_bias, norm_w, out, Hk, Hv, D, width,
               scale, eps_l2, eps_norm):
    """proj: the in-projection rows [B, N_in] (dtype of out)."""
    B = positions.shape[0]
    call("sn_gdn_decode", _p(proj), proj.stride(0), _p(conv_ring), _p(conv_w), _p(state), _p(slot_idx),
         _p(positions), _p(A_log), _p(dt_bias), _p(norm_w), _p(out), B, Hk, Hv, D, width, scale, eps_l2, eps_norm,
         dtype_code(out.dtype), _s())


def kda_decode(proj, fg, conv_ring, conv_w, state, slot_idx, positions, A_log, dt_bias, g2_b, norm_w, out, H, D,
               rank, width, scale, eps_l2, eps_norm):
    """proj: the in-projection rows [B, N_in]; fg [B, 2*H*D] = [f1 @ f2^T | g1 @ g2^T] (dtype of out)."""
    B = positions.shape[0]
    call("sn_kda_decode", _p(proj), proj.stride(0), _p(fg), _p(conv_ring), _p(conv_w), _p(state), _p(slot_idx),
         _p(positions), _p(A_log), _p(dt_bias), _p(g2_b), _p(norm_w), _p(out), B, H, D, rank, width,
         scale, eps_l2, eps_norm, dtype_code(out.dtype), _s())


def kda_gate_factors(proj, f2, g2, fg, H, D, rank, fg2=None):
    """fg [B, 2*H*D] = [f1 @ f2^T | g1 @ g2^T] from the adjacent f1 / g1 columns of the KDA
    in-projection: one decode GEMM against the block-diagonal fg2 = [f2 0; 0 g2] (2*H*D x
    2*rank, built once by the model), or two GEMMs into the two halves when fg2 is not given."""
    f1_off = 3 * H * D
    HD = H * D
    if fg2 is not None:
        gemm_decode(proj[:, f1_off:f1_off + 2 * rank], fg2, fg, "store")
        return
    gemm_decode(proj[:, f1_off:f1_off + rank], f2, fg[:, :HD], "store")
    gemm_decode(proj[:, f1_off + rank:f1_off + 2 * rank], g2, fg[:, HD:], "store")


def conv_prefill(x, x_stride, y, conv_w, conv_ring, cu_seqlens, slot_idx, channels, width, ring_hist=None,
                 pos0=None):
    call("sn_conv_prefill", _p(x), x_stride, _p(y), _p(conv_w), _p(conv_ring), _p(ring_hist), _p(cu_seqlens),
         _p(slot_idx), _p(pos0), cu_seqlens.numel() - 1, y.shape[0], channels, width, dtype_code(y.dtype), _s())


def delta_prep(kind, qkv_conv, proj, b_off, a_off, f, A_log, dt_bias, qn, kn, gexp, beta, Hk, Hv, D, scale, eps_l2,
               glog=None):
    """qn / kn: fp32 (the token scan, the KDA chunk pass) or bf16 (the chunked GDN prefill's TMA tiles)."""
    assert qn.dtype == kn.dtype
    call("sn_delta_prep", kind, _p(qkv_conv), _p(proj), proj.stride(0), b_off, a_off, _p(f), _p(A_log), _p(dt_bias),
         _p(qn), _p(kn), _p(gexp), _p(glog), _p(beta), qkv_conv.shape[0], Hk, Hv, D, scale, eps_l2,
         dtype_code(qn.dtype), dtype_code(qkv_conv.dtype), _s())


def delta_scan(kind, qn, kn, qkv_conv, v_off, gexp, beta, o, state, slot_idx, cu_seqlens, Hk, Hv, D, init_state):
    call("sn_delta_scan", kind, _p(qn), _p(kn), _p(qkv_conv), v_off, qkv_conv.stride(0), _p(gexp), _p(beta), _p(o),
         _p(state), _p(slot_idx), _p(cu_seqlens), cu_seqlens.numel() - 1, Hk, Hv, D, int(init_state),
         dtype_code(qkv_conv.dtype), _s())


def gated_rmsnorm(o, gate, gate_stride, norm_w, out, H, D, eps, act):
    call("sn_gated_rmsnorm", _p(o), _p(gate), gate_stride, _p(norm_w), _p(out), o.shape[0], H, D, eps, act,
         dtype_code(out.dtype), _s())


GEMM_MODES = {"store": SN_GEMM_STORE, "resid": SN_GEMM_RESID, "partial": SN_GEMM_PARTIAL,
              "swiglu_il": SN_GEMM_SWIGLU_IL, "attn_in": SN_GEMM_ATTN_IN}


def gemm_swiglu_block(N):
    """Block half-height h of the interleaved SwiGLU weight layout (mode "swiglu_il")."""
    return _lib.load().sn_gemm_swiglu_block(N)


def rope_pair_interleave(w_qkv, Hq, Hkv, D):
    """Reorder the q and k rows of every head of a fused [q | k | v] projection weight so that
    rotary partners sit next to each other (row 2i = dim i, row 2i+1 = dim i + D/2); v rows
    unchanged.  The decode in-projection (mode "attn_in") and the prefill RoPE (pair_il=True)
    read this order."""
    half = D // 2
    perm = torch.arange(D).view(2, half).t().reshape(-1)  # [0, D/2, 1, D/2+1, ...]
    idx = torch.cat([h * D + perm for h in range(Hq + Hkv)] + [torch.arange((Hq + Hkv) * D, (Hq + 2 * Hkv) * D)])
    return w_qkv[idx.to(w_qkv.device)].contiguous()


def interleave_swiglu(w_gu, h):
    """[gate; up] ([2N, K]) -> blocks of h gate rows then the same h up rows, zero-padded to
    ceil(N / h) blocks of 2h rows: the weight layout of mode "swiglu_il"."""
    N2, K = w_gu.shape
    N = N2 // 2
    nb = -(-N // h)
    out = torch.zeros(nb * 2 * h, K, dtype=w_gu.dtype, device=w_gu.device)
    i = torch.arange(N, device=w_gu.device)
    dst = (i // h) * (2 * h) + i % h
    out.index_copy_(0, dst, w_gu[:N])
    out.index_copy_(0, dst + h, w_gu[N:])
    return out


def deinterleave_swiglu(gu_il, N, h):
    """Inverse of interleave_swiglu on GEMM outputs: [rows, nb*2h] -> [rows, 2N] = [gate | up]."""
    rows = gu_il.shape[0]
    v = gu_il.view(rows, -1, 2, h)
    return torch.cat([v[:, :, 0].reshape(rows, -1)[:, :N], v[:, :, 1].reshape(rows, -1)[:, :N]], 1)


def gemm_decode_plan(M, N, K, mode="store"):
    """{br, splits, ks, blocks, grid, stages} the library picks for this shape (introspection)."""
    out = (ctypes.c_int * 6)()
    _lib.load().sn_gemm_decode_plan(M, N, K, GEMM_MODES.get(mode, mode), out)
    return dict(zip(("br", "splits", "ks", "blocks", "grid", "stages"), list(out)))


def gemm_decode(x, w, out, mode):
    """out (+)= x @ w.T with the decode GEMM (tcgen05 for bf16, CUDA cores for fp32); returns
    the K split count S.  x [M, K], w [N, K] (mode "swiglu_il": the interleaved [nb*2h, K]
    layout, out [M, N] = silu(g)*u); "store": out dtype [M, N]; "resid": out fp32 [M, N] +=
    x @ w.T; "partial": out fp32 [>=S, M, N] K-split slabs (slab order sums them)."""
    M, K = x.shape
    N = out.shape[-1]
    if mode == "swiglu_il":
        h = gemm_swiglu_block(N)
        assert w.shape[0] == -(-N // h) * 2 * h, "weight not in the interleaved layout for this shape"
    else:
        assert w.shape[0] == N
    assert out.dtype == (torch.float32 if mode in ("resid", "partial") else x.dtype)
    if mode == "partial":
        assert out.dim() == 3 and out.shape[1] == M and out.is_contiguous()
    assert x.dtype == w.dtype and x.stride(1) == 1 and w.stride(1) == 1 and out.stride(-1) == 1
    s_out = ctypes.c_int(1)
    call("sn_gemm_decode", _p(x), M, K, x.stride(0), _p(w), N, w.stride(0), _p(out), out.stride(-2),
         GEMM_MODES[mode], ctypes.byref(s_out), dtype_code(x.dtype), _s())
    return s_out.value


def gemm_decode_attn_in(x, w, positions, inv_freq, q_out, k_cache, v_cache, block_table, Hq, Hkv, D, page_size,
                        window, err_flag, rope_cs=None):
    """Attention in-projection with RoPE + KV append fused; w in rope_pair_interleave order;
    rope_cs: the step's (cos, sin) table from embed (default: evaluated per head)."""
    M, K = x.shape
    call("sn_gemm_decode_attn_in", _p(x), M, K, x.stride(0), _p(w), w.stride(0), _p(positions), _p(inv_freq),
         _p(q_out), _p(k_cache), _p(v_cache), _p(block_table), Hq, Hkv, D, page_size, block_table.shape[1], window,
         _p(err_flag), _p(rope_cs), dtype_code(x.dtype), _s())


def chunk_plan(cu_seqlens_host, chunk=64, device="cuda"):
    """(chunks int32 [n, 2] = (first token, length), seq_chunk0 int32 [S+1]) for the two-phase prefill."""
    chunks, starts = [], [0]
    for s0, s1 in zip(cu_seqlens_host[:-1], cu_seqlens_host[1:]):
        for t in range(int(s0), int(s1), chunk):
            chunks.append((t, min(chunk, int(s1) - t)))
        starts.append(len(chunks))
    return (torch.tensor(chunks, dtype=torch.int32, device=device).view(-1, 2),
            torch.tensor(starts, dtype=torch.int32, device=device))


def gdn_chunk_prefill2(qn, kn, qkv_conv, v_off, glog, beta, chunks, seq_chunk0, o, state, slot_idx, Hk, Hv, D,
                       init_state, workspace=None):
    n = chunks.shape[0]
    nbytes = _lib.load().sn_gdn_chunk_workspace_bytes(n, Hv, D)
    if workspace is None or workspace.numel() < nbytes:
        workspace = torch.empty(nbytes, dtype=torch.uint8, device=qn.device)
    if qn.dtype != torch.bfloat16:  # the kernel reads bf16 TMA tiles (sn_delta_prep emits them directly)
        qn, kn = qn.to(torch.bfloat16), kn.to(torch.bfloat16)
    assert qn.is_contiguous() and kn.is_contiguous()
    call("sn_gdn_chunk_prefill2", _p(qn), _p(kn), _p(qkv_conv), v_off, qkv_conv.stride(0), qkv_conv.shape[0],
         _p(glog), _p(beta),
         _p(chunks), _p(seq_chunk0), n, _p(workspace), _p(o), _p(state), _p(slot_idx), seq_chunk0.numel() - 1, Hk, Hv,
         D, int(init_state), dtype_code(qkv_conv.dtype), _s())
    return workspace



def kda_chunk_prefill2(qn, kn, qkv_conv, v_off, glog, beta, chunks, seq_chunk0, o, state, slot_idx, H, D, init_state,
                       workspace=None):
    """Two-phase chunked KDA prefill (per-channel gates glog [rows, H, D])."""
    n = chunks.shape[0]
    nbytes = _lib.load().sn_kda_chunk_workspace_bytes(n, H, D)
    if workspace is None or workspace.numel() < nbytes:
        workspace = torch.empty(nbytes, dtype=torch.uint8, device=qn.device)
    if qn.dtype != torch.bfloat16:  # the kernel reads bf16 TMA tiles (sn_delta_prep emits them directly)
        qn, kn = qn.to(torch.bfloat16), kn.to(torch.bfloat16)
    assert qn.is_contiguous() and kn.is_contiguous()
    call("sn_kda_chunk_prefill2", _p(qn), _p(kn), _p(qkv_conv), v_off, qkv_conv.stride(0), qkv_conv.shape[0],
         _p(glog), _p(beta),
         _p(chunks), _p(seq_chunk0), n, _p(workspace), _p(o), _p(state), _p(slot_idx), seq_chunk0.numel() - 1, H, D,
         int(init_state), dtype_code(qkv_conv.dtype), _s())
    return workspace


def swiglu_il(gu_il, out, ffn, h):
    """out [rows, ffn] = silu(gate) * up from the interleaved gate/up GEMM output [rows, nb*2h]."""
    call("sn_swiglu_il", _p(gu_il), gu_il.stride(0), _p(out), gu_il.shape[0], ffn, h, dtype_code(out.dtype), _s())


def tp_arrive(counter_ptr: int):
    """Bump this rank's arrival counter (after the partial product in stream order)."""
    call("sn_tp_arrive", counter_ptr, _s())


def tp_allreduce_add_rmsnorm(peer_slabs, peer_counters, world, rank, nsplit, residual, weight, out, eps):
    """residual += sum over ranks and slabs of the peers' partials (P2P), then out = RMSNorm(residual) * weight."""
    rows, dim = residual.shape
    call("sn_tp_allreduce_add_rmsnorm", _p(peer_slabs), _p(peer_counters), world, rank, nsplit, _p(residual),
         _p(weight), _p(out), rows, dim, eps, dtype_code(out.dtype), _s())


# ------------------------------------------------------------------ fused decode chain
def chain_gemm(x, w, out, mode, depends=True, ss_out=None, **attn):
    """A GEMM phase of decode_chain (see gemm_decode for the modes; attention in-projection:
    mode "attn_in" with positions, inv_freq, q_out, k_cache, v_cache, block_table, Hq, Hkv, D,
    page_size, window, err_flag)."""
    M, K = x.shape
    N = out.shape[-1] if mode != "attn_in" else (attn["Hq"] + 2 * attn["Hkv"]) * attn["D"]
    assert x.dtype == torch.bfloat16 and w.dtype == torch.bfloat16 and x.stride(1) == 1 and w.stride(1) == 1
    if mode == "swiglu_il":
        h = gemm_swiglu_block(N)
        assert w.shape[0] == -(-N // h) * 2 * h, "weight not in the interleaved layout for this shape"
    elif mode != "attn_in":
        assert w.shape[0] == N
    ph = dict(kind=SN_CHAIN_GEMM, depends=int(depends), x=_p(x), K=K, ldx=x.stride(0), w=_p(w), N=N,
              ldw=w.stride(0), mode=GEMM_MODES[mode], keep=(x, w, out))
    if mode == "attn_in":
        bt = attn["block_table"]
        ph.update(out=attn["q_out"].data_ptr(), ldo=0, positions=_p(attn["positions"]),
                  inv_freq=_p(attn["inv_freq"]), q_out=_p(attn["q_out"]), k_cache=_p(attn["k_cache"]),
                  v_cache=_p(attn["v_cache"]), block_table=_p(bt), Hq=attn["Hq"], Hkv=attn["Hkv"], D=attn["D"],
                  page_size=attn["page_size"], max_blocks=bt.shape[1], window=attn["window"],
                  err_flag=_p(attn.get("err_flag")), rope_cs=_p(attn.get("rope_cs")))
    else:
        assert out.dtype == (torch.float32 if mode in ("resid", "partial") else torch.bfloat16)
        if mode == "partial":
            assert out.dim() == 3 and out.shape[1] == M and out.is_contiguous()
        ph.update(out=_p(out), ldo=out.stride(-2))
    if ss_out is not None:
        assert mode == "resid" and ss_out.dtype == torch.float32 and ss_out.is_contiguous()
        ph.update(ss_out=_p(ss_out))
    return ph


def chain_norm(residual, weight, out, eps, partials=None, nsplit=-1, ss_in=None, n_ss=-1, depends=True):
    """A NORM phase: residual += sum of the slabs (nsplit < 0: the splits of the latest PARTIAL
    GEMM phase before it); out = rmsnorm(residual) * weight.  ss_in: take each row's sum of
    squares from the per-block sums a RESID GEMM phase wrote (n_ss < 0: its block count)."""
    assert residual.dtype == torch.float32 and residual.is_contiguous() and out.dtype == torch.bfloat16
    if partials is None:
        nsplit = 0
    if ss_in is None:
        n_ss = 0
    return dict(kind=SN_CHAIN_NORM, depends=int(depends), partials=_p(partials), nsplit=nsplit,
                residual=_p(residual), weight=_p(weight), norm_out=_p(out), dim=residual.shape[1], eps=float(eps),
                ss_in=_p(ss_in), n_ss=n_ss, keep=(residual, weight, out, partials, ss_in))


def decode_chain(phases, M, counter):
    """Run the phases (chain_gemm / chain_norm dicts) as one persistent launch; counter: an
    int64 device word for this call site (zero-initialised once, never reset).  Returns the K
    split count of every phase (PARTIAL GEMMs and the norms that consume them)."""
    n = len(phases)
    arr = (ChainPhase * n)()
    for i, ph in enumerate(phases):
        for k, v in ph.items():
            if k != "keep":
                setattr(arr[i], k, v)
    assert counter.dtype == torch.int64 and counter.is_cuda
    call("sn_decode_chain", ctypes.cast(arr, ctypes.c_void_p), n, M, _p(counter), _s())
    return [arr[i].splits for i in range(n)]


# ------------------------------------------------------------------ prefill GEMM
def gemm_prefill(a, w, out=None, swiglu_h=0):
    """out [M, N] = a [M, K] @ w [N, K]^T (bf16 operands, tcgen05; out bf16, or fp32 when an
    fp32 out is given).  swiglu_h > 0: w is the SwiGLU-interleaved gate/up layout
    (interleave_swiglu, block swiglu_h) and out [M, F] = silu(gate) * up with F = the FFN width
    (out must be given)."""
    M, K = a.shape
    assert a.dtype == torch.bfloat16 and w.dtype == torch.bfloat16 and a.stride(1) == 1 and w.stride(1) == 1
    if swiglu_h:
        assert out is not None
        N = out.shape[1]
        assert w.shape[0] == -(-N // swiglu_h) * 2 * swiglu_h
    else:
        N = w.shape[0]
        if out is None:
            out = torch.empty(M, N, device=a.device, dtype=torch.bfloat16)
    f32 = out.dtype == torch.float32
    assert (out.dtype == torch.bfloat16 or (f32 and not swiglu_h)) and out.stride(1) == 1 and out.shape[0] == M
    mode = SN_GEMM_SWIGLU_IL if swiglu_h else (GEMM_MODES["partial"] if f32 else SN_GEMM_STORE)
    call("sn_gemm_prefill", _p(a), M, K, a.stride(0), _p(w), N, w.stride(0), _p(out), out.stride(0), mode,
         swiglu_h, _s())
    return out
