"""Placement-driven supernet runtime: layer loop, heterogeneous state pools,
prefill and decode — the host side of the mixer step.

Paper mapping:
  * one mixer per layer chosen by the placement (R/PAPER.md:860-865); the layer
    loop launches only that mixer's kernels, keyed by the immutable table
    `self.kinds` (no global mutable state, so several Supernet objects — one per
    placement — can share a process and a GPU);
  * heterogeneous state (R/PAPER.md:834-843): FA paged KV, SWA ring KV, GDN/KDA
    fp32 recurrent state + conv ring — here separate pools per mixer kind, sized
    exactly, instead of vLLM's unified page size padding (which the paper blames
    for its hybrid overhead, R/PAPER.md:1797, 1804);
  * dual execution path (R/PAPER.md:845-850): a parallel prefill over the whole
    prompt, then one fused in-place decode step per token;
  * CUDA graphs per placement (R/PAPER.md:831, 863): see graphs.py.

All compute runs in libsn100.so kernels (ops.py) plus cuBLAS GEMMs for the
projections / FFN / LM head; there is no CPU path.
"""
from __future__ import annotations

import math

import torch

from . import ops
from ._lib import load as _load_lib
from .config import SupernetConfig, attn_scale
from .placement import FA, GDN, KDA, SWA, layer_kinds
from .weights import cast_weights, init_weights


def _ceil(a, b):
    return (a + b - 1) // b


def choose_split(max_pages: int, rows: int, sms: int = 148, cap: int = 64, floor: int = 4,
                 per_sm: int | None = None) -> tuple[int, int]:
    """Split-KV decomposition for decode attention: aim for ~4 CTAs per SM over
    (sequence x kv head x split); returns (split_pages, max_splits).  A split gets at least
    `floor` pages (every warp of the CTA streams >= 2 tiles) unless the sequence is shorter:
    with one-page splits at B=1 the CTAs were mostly setup and the last CTA's merge over 64
    partials dominated (SWA decode 59 us/layer at B=1, tools/ablate.py).  The bf16 kernel holds
    one CTA per SM (196 KB of TMA stages), so with fewer (sequence x kv head) rows than SMs the
    splits fill exactly one wave (all-FA B=1: 8.78 -> 7.51 ms/step at 32K, 11.6 -> 10.3 at 128K);
    with more, ~4 CTAs per SM balance the tail."""
    if per_sm is None:
        per_sm = 1 if rows < sms else 4
    want = max(1, _ceil(per_sm * sms, max(rows, 1)))
    split_pages = max(1, min(cap, max(min(floor, max_pages), _ceil(max_pages, want))))
    return split_pages, _ceil(max_pages, split_pages)


class Supernet:
    """A loaded placement of the supernet with its state pools.

    placement: code string ("ASKG..."), list of type names, or a
    placeopt-compatible Placement.  weights: optional pre-built structure
    (paper_2604_19877_b200.weights.init_weights); default is the seeded random
    init generated directly on the device.
    """

    def __init__(self, cfg: SupernetConfig, placement, *, batch: int, max_len: int, dtype=torch.bfloat16,
                 device="cuda", seed: int = 0, weights=None, fa_block_table=None, tp_group=None,
                 tp_transport: str = "p2p", fused_chain: bool = False):
        _load_lib()  # fail loudly if the extension is missing
        self.B, self.max_len, self.dtype = batch, max_len, dtype
        self.device = torch.device(device)
        if self.device.type != "cuda":
            raise ValueError("Supernet runs on CUDA only (no CPU fallback)")
        self.kinds = layer_kinds(placement)
        if len(self.kinds) != cfg.num_layers:
            raise ValueError(f"placement has {len(self.kinds)} layers, config {cfg.name} has {cfg.num_layers}")
        if weights is None:
            weights = init_weights(cfg, self.kinds, seed=seed, device=self.device, dtype=dtype)
        # head-parallel tensor parallelism (dist.py): local head counts, sharded weights, one
        # all-reduce after each mixer out-projection and after each FFN down-projection
        self.tp_group, self.tp = tp_group, 1
        if tp_group is not None:
            import torch.distributed as tdist
            from .dist import shard_weights, tp_config
            self.tp, rank = tdist.get_world_size(tp_group), tdist.get_rank(tp_group)
            if self.tp > 1:
                weights = shard_weights(cfg, self.kinds, weights, self.tp, rank)
                cfg = tp_config(cfg, self.tp)
        self.cfg = cfg
        self._fused_chain = fused_chain
        self.w = cast_weights(weights, self.device, dtype)
        del weights  # self.w may alias it; the FFN interleave below must free the original rows
        self.inv_freq = cfg.inv_freq().to(device=self.device, dtype=torch.float32)
        self.scale_attn = attn_scale(cfg)
        self._alloc_state(fa_block_table)
        self._alloc_decode_buffers()
        # head-parallel decode: the row-parallel all-reduces run through peer memory (CUDA IPC,
        # NVLink P2P), fused into the next residual add + RMSNorm (csrc/sn_tp.cu) — "p2p", one
        # process per GPU on a node — or through NCCL ("nccl": any transport NCCL has)
        if tp_transport not in ("p2p", "nccl"):
            raise ValueError(f"tp_transport {tp_transport!r}: 'p2p' or 'nccl'")
        self.sym = None
        if self.tp > 1 and tp_transport == "p2p":
            from .dist import SymmetricSlabs
            self.sym = SymmetricSlabs(batch, cfg.hidden, group=tp_group, device=self.device)

        self.probe = None  # optional KernelProbe: CUDA events around the mixer kernels (bench instrumentation)
        # every decode projection runs on the library's decode GEMM (tcgen05 for bf16, the CUDA-core
        # tile kernel for the fp32 numerics mode); the gate/up rows are interleaved in blocks of h
        # (SwiGLU fused into the GEMM epilogue: one contiguous weight stream, no [gate; up] copy) and
        # the attention q / k rows in rotary pairs (RoPE + KV append fused into the in-projection)
        ffn = self.cfg.ffn
        hb = ops.gemm_swiglu_block(ffn)
        self.gu_il = (ffn, hb)
        for lw in self.w["layers"]:
            if "ffn_gu_il" in lw:  # prebuilt and shared (serving.SupernetStore), tagged with its block
                if lw.get("ffn_gu_hb") != hb:
                    raise ValueError(f"prebuilt SwiGLU-interleaved FFN weights use block {lw.get('ffn_gu_hb')}, "
                                     f"this engine needs {hb}")
            else:
                lw["ffn_gu_il"] = ops.interleave_swiglu(lw.pop("ffn_gu"), hb)
                lw["ffn_gu_hb"] = hb
        for l, kind in enumerate(self.kinds):
            mw = self.w["layers"][l]["mixer"]
            if kind in (FA, SWA) and "qkv_il" not in mw:
                mw["qkv_il"] = ops.rope_pair_interleave(mw.pop("qkv"), cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim)
            if kind == KDA and "fg2" not in mw:  # the two low-rank gate factors as one decode GEMM
                mw["fg2"] = torch.block_diag(mw["f2"], mw["g2"]).contiguous()

    # ------------------------------------------------------------------ state pools
    def _alloc_state(self, fa_block_table):
        cfg, B, dev, dt = self.cfg, self.B, self.device, self.dtype
        P, Hkv, D = cfg.page_size, cfg.n_kv_heads, cfg.head_dim
        i32 = dict(device=dev, dtype=torch.int32)
        self.seq_lens = torch.zeros(B, **i32)
        self.positions = torch.zeros(B, **i32)
        self.fa_blocks = _ceil(self.max_len, P)
        if fa_block_table is None:
            fa_block_table = torch.arange(B * self.fa_blocks, dtype=torch.int32).view(B, self.fa_blocks)
        self.fa_block_table = fa_block_table.to(**i32).contiguous()
        self.fa_pages = int(self.fa_block_table.max().item()) + 1 if self.fa_block_table.numel() else 0
        if cfg.window % P:
            raise ValueError("SWA window must be a multiple of the page size")
        self.swa_blocks = cfg.window // P
        self.swa_block_table = torch.arange(B * self.swa_blocks, **i32).view(B, self.swa_blocks)
        self.state = []
        for kind in self.kinds:
            if kind == FA:
                shape = (self.fa_pages, Hkv, P, D)
                self.state.append({"k": torch.zeros(shape, device=dev, dtype=dt),
                                   "v": torch.zeros(shape, device=dev, dtype=dt)})
            elif kind == SWA:
                shape = (B * self.swa_blocks, Hkv, P, D)
                self.state.append({"k": torch.zeros(shape, device=dev, dtype=dt),
                                   "v": torch.zeros(shape, device=dev, dtype=dt)})
            elif kind == GDN:
                Dg = cfg.gdn_head_dim
                self.state.append({"S": torch.zeros(B, cfg.gdn_v_heads, Dg, Dg, device=dev, dtype=torch.float32),
                                   "conv": torch.zeros(B, cfg.gdn_conv_channels, cfg.conv_width, device=dev, dtype=dt)})
            else:
                Dk = cfg.kda_head_dim
                self.state.append({"S": torch.zeros(B, cfg.kda_heads, Dk, Dk, device=dev, dtype=torch.float32),
                                   "conv": torch.zeros(B, cfg.kda_conv_channels, cfg.conv_width, device=dev, dtype=dt)})

    def reset(self):
        self.seq_lens.zero_()
        for st in self.state:
            for t in st.values():
                t.zero_()

    def state_bytes(self) -> int:
        return sum(t.numel() * t.element_size() for st in self.state for t in st.values())

    def weight_bytes(self) -> int:
        def walk(o):
            if isinstance(o, dict):
                return sum(walk(v) for v in o.values())
            if isinstance(o, list):
                return sum(walk(v) for v in o)
            return o.numel() * o.element_size() if torch.is_tensor(o) else 0
        return walk(self.w)

    # ------------------------------------------------------------------ decode buffers
    def _alloc_decode_buffers(self):
        cfg, B, dev, dt = self.cfg, self.B, self.device, self.dtype
        e = lambda *s, d=dt: torch.empty(*s, device=dev, dtype=d)
        self.step_tokens = torch.zeros(B, device=dev, dtype=torch.int32)
        self.next_tokens = torch.zeros(B, device=dev, dtype=torch.int32)
        self.residual = e(B, cfg.hidden, d=torch.float32)
        self.h = e(B, cfg.hidden)
        self.mix_out = e(B, cfg.hidden)
        self.ffn_out = e(B, cfg.hidden)
        self.gu = e(B, 2 * cfg.ffn)
        self.act = e(B, cfg.ffn)
        self.logits = e(B, cfg.vocab)
        self.err_flag = torch.zeros(1, device=dev, dtype=torch.int32)  # KV append past the block table
        # fused decode chains (bf16, one GPU): one grid-barrier counter per call site, on its own
        # 64-byte line; zeroed once, never reset (csrc/sn_chain.cu)
        # Measured (profiles/r02_chain.md): 10.47 ms/step fused vs 10.22 separate at B=64 / 32K —
        # each grid-wide norm dependency costs ~5 us of L2 round trips under full HBM load, more
        # than the kernel boundaries it removes; off by default, kept under test.
        self.use_chain = bool(self._fused_chain) and dt == torch.bfloat16 and self.tp == 1 and B <= 128
        self.chain_ctr = torch.zeros(len(self.kinds) + 1, 8, device=dev, dtype=torch.int64)[:, 0]
        # fp32 K-split slabs of the residual-updating projections (o-proj, FFN down), summed into
        # the residual in slab order by the next add + RMSNorm
        self.slab = e(8, B, cfg.hidden, d=torch.float32)
        kinds = set(self.kinds)
        self.dec = {}
        if kinds & {FA, SWA}:
            Hq, Hkv, D = cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim
            self.dec["q"] = e(B, Hq, D)
            self.dec["attn"] = e(B, Hq * D)
            self.dec["counters"] = torch.zeros(B * Hkv, device=dev, dtype=torch.int32)
            # the step's rotary (cos, sin) per (slot, pair), written by the embed kernel
            self.dec["rope_cs"] = e(B, D // 2, 2, d=torch.float32)
            self.attn_split = {}
            for kind, max_keys in ((FA, self.max_len), (SWA, cfg.window)):
                if kind in kinds:
                    self.attn_split[kind] = choose_split(_ceil(max_keys, cfg.page_size), B * Hkv)
            ms_max = max(ms for _, ms in self.attn_split.values())
            nbytes = ops.attn_decode_workspace_bytes(B, Hq, Hkv, D, ms_max)
            self.dec["ws"] = torch.empty(max(nbytes // 4, 1), device=dev, dtype=torch.float32)
            self.ws_max_splits = ms_max
        # in-projection rows padded to 16 bytes (TMA row pitch of the gate-factor GEMMs' operand)
        pad8 = lambda n: -(-n // 8) * 8
        if GDN in kinds:
            self.dec["gdn_proj"] = e(B, pad8(cfg.gdn_in_width))[:, :cfg.gdn_in_width]
            self.dec["gdn_out"] = e(B, cfg.gdn_value_dim)
        if KDA in kinds:
            self.dec["kda_proj"] = e(B, pad8(cfg.kda_in_width))[:, :cfg.kda_in_width]
            self.dec["kda_out"] = e(B, cfg.kda_dim)
            self.dec["kda_fg"] = e(B, 2 * cfg.kda_dim)  # [f | g] per row

    # ------------------------------------------------------------------ decode
    def _gemm(self, x, w, out, mode, role):
        self._probe_begin("gemm_" + role, fine=True)
        ns = ops.gemm_decode(x, w, out, mode)
        self._probe_end("gemm_" + role, fine=True)
        return ns

    def _attn_decode(self, l, kind, h):
        cfg, st, w, d = self.cfg, self.state[l], self.w["layers"][l]["mixer"], self.dec
        Hq, Hkv, D, P = cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim, cfg.page_size
        window = cfg.window if kind == SWA else 0
        bt = self.swa_block_table if kind == SWA else self.fa_block_table
        # in-projection with RoPE + the KV append fused into its epilogue
        self._probe_begin("gemm_in_proj", fine=True)
        ops.gemm_decode_attn_in(h, w["qkv_il"], self.positions, self.inv_freq, d["q"], st["k"], st["v"], bt, Hq, Hkv,
                                D, P, window, self.err_flag, rope_cs=d["rope_cs"])
        self._probe_end("gemm_in_proj", fine=True)
        sp, _ = self.attn_split[kind]
        name = "swa_decode" if kind == SWA else "fa_decode"
        self._probe_begin(name)
        ops.attn_decode(d["q"], st["k"], st["v"], bt, self.seq_lens, d["attn"], d["ws"], d["counters"], Hq, Hkv, D,
                        P, window, sp, self.ws_max_splits, self.scale_attn)
        self._probe_end(name)
        return self._residual_proj(d["attn"], w["o"], "out_proj")

    def _gdn_decode(self, l, h):
        cfg, st, w, d = self.cfg, self.state[l], self.w["layers"][l]["mixer"], self.dec
        D = cfg.gdn_head_dim
        self._gemm(h, w["w_in"], d["gdn_proj"], "store", "in_proj")
        self._probe_begin("gdn_decode")
        ops.gdn_decode(d["gdn_proj"], st["conv"], w["conv_w"], st["S"], None, self.positions, w["A_log"],
                       w["dt_bias"], w["norm_w"], d["gdn_out"], cfg.gdn_k_heads, cfg.gdn_v_heads, D, cfg.conv_width,
                       1.0 / math.sqrt(D), cfg.l2_eps, cfg.mixer_norm_eps)
        self._probe_end("gdn_decode")
        return self._residual_proj(d["gdn_out"], w["o"], "out_proj")

    def _kda_decode(self, l, h):
        cfg, st, w, d = self.cfg, self.state[l], self.w["layers"][l]["mixer"], self.dec
        D = cfg.kda_head_dim
        self._gemm(h, w["w_in"], d["kda_proj"], "store", "in_proj")
        self._probe_begin("kda_gates", fine=True)
        ops.kda_gate_factors(d["kda_proj"], w["f2"], w["g2"], d["kda_fg"], cfg.kda_heads, D, cfg.kda_rank,
                             fg2=w["fg2"])
        self._probe_end("kda_gates", fine=True)
        self._probe_begin("kda_decode")
        ops.kda_decode(d["kda_proj"], d["kda_fg"], st["conv"], w["conv_w"], st["S"], None, self.positions, w["A_log"],
                       w["dt_bias"], w["g2_b"], w["norm_w"], d["kda_out"], cfg.kda_heads, D, cfg.kda_rank,
                       cfg.conv_width, 1.0 / math.sqrt(D), cfg.l2_eps, cfg.mixer_norm_eps)
        self._probe_end("kda_decode")
        return self._residual_proj(d["kda_out"], w["o"], "out_proj")

    def _probe_begin(self, name, fine=False):
        if self.probe is not None and (self.probe.fine or not fine):
            self.probe.begin(name)

    def _probe_end(self, name, fine=False):
        if self.probe is not None and (self.probe.fine or not fine):
            self.probe.end(name)

    def _residual_proj(self, x, w, role):
        """A projection whose result is added to the residual stream: fp32 K-split slabs that the
        next add + RMSNorm sums in slab order.  Head-parallel: this rank's row-parallel partial
        slabs go through the all-reduce first (peer memory, fused into that norm; or NCCL).
        Returns the (transport, slabs, nsplit) the next _norm() takes."""
        if self.sym is not None:  # partial straight into this rank's symmetric slabs (peer memory)
            parity = 0 if role == "out_proj" else 1
            ns = self._gemm(x, w, self.sym.local_slabs(parity), "partial", role)
            ops.tp_arrive(self.sym.counter_ptr())
            return ("p2p", parity, ns)
        ns = self._gemm(x, w, self.slab, "partial", role)
        if self.tp > 1:  # NCCL transport: the partial slabs are summed over the group first
            from .dist import allreduce_sum_
            allreduce_sum_(self.slab[:ns], self.tp_group)
        return ("local", self.slab, ns)

    def _norm(self, pending, weight):
        self._probe_begin("add_rmsnorm", fine=True)
        if pending is None:
            ops.add_rmsnorm(None, self.residual, weight, self.h, self.cfg.norm_eps)
        elif pending[0] == "p2p":
            sym = self.sym
            ops.tp_allreduce_add_rmsnorm(sym.slab_ptrs[pending[1]], sym.counters, sym.world, sym.rank, pending[2],
                                         self.residual, weight, self.h, self.cfg.norm_eps)
        else:
            ops.add_rmsnorm(None, self.residual, weight, self.h, self.cfg.norm_eps, partials=pending[1],
                            nsplit=pending[2])
        self._probe_end("add_rmsnorm", fine=True)

    def decode_body(self):
        """One decode step on the current stream: step_tokens -> logits, next_tokens.
        Graph-capturable: every size/position it needs is read from device buffers."""
        if self.use_chain:
            return self._decode_body_chain()
        w = self.w
        self._probe_begin("embed", fine=True)
        ops.embed(self.step_tokens, w["embed"], self.residual, self.seq_lens, self.positions, self.inv_freq,
                  self.dec.get("rope_cs"))
        self._probe_end("embed", fine=True)
        pending = None
        for l, kind in enumerate(self.kinds):
            lw = w["layers"][l]
            self._norm(pending, lw["norm1"])
            if kind == GDN:
                pending = self._gdn_decode(l, self.h)
            elif kind == KDA:
                pending = self._kda_decode(l, self.h)
            else:
                pending = self._attn_decode(l, kind, self.h)
            self._norm(pending, lw["norm2"])
            self._gemm(self.h, lw["ffn_gu_il"], self.act, "swiglu_il", "ffn_gate_up")
            pending = self._residual_proj(self.act, lw["ffn_down"], "ffn_down")
        self._norm(pending, w["final_norm"])
        self._gemm(self.h, w["lm_head"], self.logits, "store", "lm_head")
        self._probe_begin("argmax", fine=True)
        ops.argmax(self.logits, self.next_tokens, self.positions)
        self._probe_end("argmax", fine=True)

    # ------------------------------------------------------------------ fused decode chain
    def _in_proj_phases(self, l):
        """Chain phases of layer l's mixer in-projection (the rows its mixer kernel reads)."""
        cfg, kind, st, d = self.cfg, self.kinds[l], self.state[l], self.dec
        w = self.w["layers"][l]["mixer"]
        if kind in (FA, SWA):
            return [ops.chain_gemm(self.h, w["qkv_il"], None, "attn_in", positions=self.positions,
                                   inv_freq=self.inv_freq, q_out=d["q"], k_cache=st["k"], v_cache=st["v"],
                                   block_table=self.swa_block_table if kind == SWA else self.fa_block_table,
                                   Hq=cfg.n_q_heads, Hkv=cfg.n_kv_heads, D=cfg.head_dim, page_size=cfg.page_size,
                                   window=cfg.window if kind == SWA else 0, err_flag=self.err_flag,
                                   rope_cs=d["rope_cs"])]
        if kind == GDN:
            return [ops.chain_gemm(self.h, w["w_in"], d["gdn_proj"], "store")]
        H, D, R = cfg.kda_heads, cfg.kda_head_dim, cfg.kda_rank
        proj, f1 = d["kda_proj"], 3 * H * D
        return [ops.chain_gemm(self.h, w["w_in"], proj, "store"),
                ops.chain_gemm(proj[:, f1:f1 + 2 * R], w["fg2"], d["kda_fg"], "store")]

    def _mixer_decode(self, l):
        """Layer l's mixer kernel (its in-projection ran at the end of the previous chain)."""
        cfg, kind, st, d = self.cfg, self.kinds[l], self.state[l], self.dec
        w = self.w["layers"][l]["mixer"]
        if kind in (FA, SWA):
            window = cfg.window if kind == SWA else 0
            bt = self.swa_block_table if kind == SWA else self.fa_block_table
            sp, _ = self.attn_split[kind]
            name = "swa_decode" if kind == SWA else "fa_decode"
            self._probe_begin(name)
            ops.attn_decode(d["q"], st["k"], st["v"], bt, self.seq_lens, d["attn"], d["ws"], d["counters"],
                            cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim, cfg.page_size, window, sp,
                            self.ws_max_splits, self.scale_attn)
            self._probe_end(name)
            return d["attn"]
        if kind == GDN:
            D = cfg.gdn_head_dim
            self._probe_begin("gdn_decode")
            ops.gdn_decode(d["gdn_proj"], st["conv"], w["conv_w"], st["S"], None, self.positions, w["A_log"],
                           w["dt_bias"], w["norm_w"], d["gdn_out"], cfg.gdn_k_heads, cfg.gdn_v_heads, D,
                           cfg.conv_width, 1.0 / math.sqrt(D), cfg.l2_eps, cfg.mixer_norm_eps)
            self._probe_end("gdn_decode")
            return d["gdn_out"]
        D = cfg.kda_head_dim
        self._probe_begin("kda_decode")
        ops.kda_decode(d["kda_proj"], d["kda_fg"], st["conv"], w["conv_w"], st["S"], None, self.positions,
                       w["A_log"], w["dt_bias"], w["g2_b"], w["norm_w"], d["kda_out"], cfg.kda_heads, D,
                       cfg.kda_rank, cfg.conv_width, 1.0 / math.sqrt(D), cfg.l2_eps, cfg.mixer_norm_eps)
        self._probe_end("kda_decode")
        return d["kda_out"]

    def _chain(self, site, phases):
        self._probe_begin("chain")
        ops.decode_chain(phases, self.B, self.chain_ctr[site])
        self._probe_end("chain")

    def _decode_body_chain(self):
        """bf16 single-GPU decode step as 1 + 2L + 2 launches: embed, then per layer one fused
        chain (out-proj -> add+RMSNorm -> FFN gate/up -> down -> add+RMSNorm -> next in-proj,
        csrc/sn_chain.cu) and the layer's mixer kernel, then argmax."""
        w, cfg, L = self.w, self.cfg, len(self.kinds)
        layers = w["layers"]
        self._probe_begin("embed", fine=True)
        ops.embed(self.step_tokens, w["embed"], self.residual, self.seq_lens, self.positions, self.inv_freq,
                  self.dec.get("rope_cs"))
        self._probe_end("embed", fine=True)
        self._chain(0, [ops.chain_norm(self.residual, layers[0]["norm1"], self.h, cfg.norm_eps)]
                    + self._in_proj_phases(0))
        for l in range(L):
            lw = layers[l]
            mix = self._mixer_decode(l)
            # the residual projections add straight into the residual stream (one writer per
            # element, no split-K slabs) and leave per-block row sums of squares for the norm
            # residual projections: fp32 split-K slabs (PARTIAL) that the next NORM phase adds to
            # the residual in slab order.  (RESID straight into the residual with per-block
            # sums of squares for the norm was measured slower: the S=1 plans leave fewer weight
            # bytes in flight per SM — 10.06 vs 9.13 ms/step, profiles/r02_chain.md.)
            rp = lambda x, wt: ops.chain_gemm(x, wt, self.slab, "partial")
            nm = lambda wt: ops.chain_norm(self.residual, wt, self.h, cfg.norm_eps, partials=self.slab)
            ph = [rp(mix, lw["mixer"]["o"]), nm(lw["norm2"]),
                  ops.chain_gemm(self.h, lw["ffn_gu_il"], self.act, "swiglu_il"),
                  rp(self.act, lw["ffn_down"])]
            if l + 1 < L:
                ph += [nm(layers[l + 1]["norm1"])] + self._in_proj_phases(l + 1)
            else:
                ph += [nm(w["final_norm"]), ops.chain_gemm(self.h, w["lm_head"], self.logits, "store")]
            self._chain(l + 1, ph)
        self._probe_begin("argmax", fine=True)
        ops.argmax(self.logits, self.next_tokens, self.positions)
        self._probe_end("argmax", fine=True)

    def kernels_per_step(self) -> dict:
        """Launch census of one decode step (all libsn100 kernels; the decode step launches no
        library GEMMs).  NCCL all-reduces of the head-parallel NCCL transport are counted apart."""
        if self.use_chain:  # embed, L + 1 chains, L mixer kernels, argmax
            return {"sn": 2 * len(self.kinds) + 3, "cublas": 0, "nccl": 0}
        sn = 4                                     # embed, final norm, LM head, argmax
        for kind in self.kinds:
            sn += 2 + 4 + 1 + (1 if kind == KDA else 0)  # norms, in/out-proj, gate/up, down, mixer (+KDA gates GEMM)
        nccl = 2 * len(self.kinds) if (self.tp > 1 and self.sym is None) else 0
        return {"sn": sn + (2 * len(self.kinds) if self.sym is not None else 0), "cublas": 0, "nccl": nccl}

    def check_capacity(self, steps: int = 1):
        """Raise before a decode that would take a sequence past max_len (its KV append would
        fall off the block table; the kernels skip such writes and set err_flag)."""
        top = int(self.seq_lens.max().item()) if self.B else 0
        if top + steps > self.max_len:
            raise ValueError(f"decode of {steps} step(s) would exceed max_len={self.max_len} (longest sequence {top})")
        if int(self.err_flag.item()):
            raise RuntimeError("a KV append fell outside the block table (err_flag set)")

    @torch.no_grad()
    def decode(self, tokens):
        """Eager decode step.  tokens: [B] ints (any device) -> logits [B, V] (device buffer)."""
        self.check_capacity()
        self.step_tokens.copy_(torch.as_tensor(tokens, dtype=torch.int32))
        self.decode_body()
        return self.logits

    # ------------------------------------------------------------------ prefill
    @torch.no_grad()
    def prefill(self, tokens, return_all: bool = False, slots=None, append: bool = False):
        """Parallel prefill from an empty state.  tokens: [B, T] (equal-length prompts) or a list
        of 1-D prompts of any lengths (ragged: packed rows, cu_seqlens, every kernel masks or
        chunks per sequence).  slots: engine batch slots the prompts go to (continuous
        batching: only those slots are reset and prefilled — their KV pages, rings, conv tails
        and recurrent states are addressed through slot indices — while the other slots keep
        decoding); default all B slots.  append: continue those sequences instead of starting
        them (chunked prefill of long prompts, multi-turn): positions start at their current
        lengths, attention also reads the cached prefix, the conv rings and recurrent states
        carry over.  Returns the last position's logits [n, V], or with return_all [n, T, V]
        (equal lengths) / a list of [T_b, V] (ragged)."""
        cfg, w, dev, dt = self.cfg, self.w, self.device, self.dtype
        ragged = isinstance(tokens, (list, tuple))
        if ragged:
            seqs = [torch.as_tensor(t).reshape(-1).to(device=dev, dtype=torch.int32) for t in tokens]
            lens = [int(t.numel()) for t in seqs]
            flat = torch.cat(seqs)
        else:
            t2 = torch.as_tensor(tokens).to(device=dev, dtype=torch.int32)
            lens = [t2.shape[1]] * t2.shape[0]
            flat = t2.reshape(-1)
        B = len(lens)
        if slots is None:
            if B != self.B:
                raise ValueError(f"prefill batch {B} != engine batch {self.B}")
            slot_list = list(range(B))
        else:
            slot_list = [int(x) for x in slots]
            if len(slot_list) != B or len(set(slot_list)) != B or not all(0 <= x < self.B for x in slot_list):
                raise ValueError(f"slots {slot_list} must be {B} distinct indices in [0, {self.B})")
        pos0 = [int(x) for x in self.seq_lens[slot_list].tolist()] if append else [0] * B
        if min(lens) < 1 or max(p + L for p, L in zip(pos0, lens)) > self.max_len:
            raise ValueError(f"prompt lengths must be >= 1 and fit max_len={self.max_len}")
        rows = sum(lens)
        i32 = dict(device=dev, dtype=torch.int32)
        cu_host = [0]
        for L in lens:
            cu_host.append(cu_host[-1] + L)
        self._cu_host = cu_host
        cu = torch.tensor(cu_host, **i32)
        lens_t = torch.tensor(lens, **i32)
        slot_t = torch.tensor(slot_list, **i32)
        self._slot_idx = None if slots is None else slot_t  # identity mapping: kernels take NULL
        pos0_t = torch.tensor(pos0, **i32)
        self._append = (pos0, pos0_t) if append else None
        row_seq = torch.repeat_interleave(slot_t, lens_t)
        row_pos = (torch.arange(rows, **i32) - torch.repeat_interleave(cu[:-1], lens_t)
                   + torch.repeat_interleave(pos0_t, lens_t))
        T = max(lens)
        if append:
            self.seq_lens.index_copy_(0, slot_t.long(), pos0_t + lens_t)
        elif slots is None:
            self.reset()
            self.seq_lens.copy_(lens_t)
        else:
            idx = slot_t.long()
            for st in self.state:
                for key in ("S", "conv"):
                    if key in st:
                        st[key].index_fill_(0, idx, 0)
            self.seq_lens.index_copy_(0, idx, lens_t)
        e = lambda *s, d=dt: torch.empty(*s, device=dev, dtype=d)
        resid = e(rows, cfg.hidden, d=torch.float32)
        # tensor parallel: the row-parallel projections (out-proj, FFN down) leave fp32 partials
        # that are summed over the group in fp32 and added to the residual before the norm
        rp_dt = torch.float32 if self.tp > 1 else dt
        h, mix, ffn_o = e(rows, cfg.hidden), e(rows, cfg.hidden, d=rp_dt), e(rows, cfg.hidden, d=rp_dt)

        def add_norm(delta, weight):
            if delta is not None and delta.dtype != h.dtype:
                resid.add_(delta)
                delta = None
            ops.add_rmsnorm(delta, resid, weight, h, cfg.norm_eps)

        ops.embed(flat, w["embed"], resid)
        delta = None
        for l, kind in enumerate(self.kinds):
            lw = w["layers"][l]
            add_norm(delta, lw["norm1"])
            if kind in (FA, SWA):
                self._attn_prefill(l, kind, h, mix, cu, row_seq, row_pos)
            elif kind == GDN:
                self._gdn_prefill(l, h, mix, cu)
            else:
                self._kda_prefill(l, h, mix, cu)
            self._tp_sum(mix)
            add_norm(mix, lw["norm2"])
            act = e(rows, cfg.ffn)
            self._mm(h, lw["ffn_gu_il"], act, swiglu=True)
            self._mm(act, lw["ffn_down"], ffn_o)
            self._tp_sum(ffn_o)
            delta = ffn_o
        add_norm(delta, w["final_norm"])
        if return_all:
            logits = self._mm(h, w["lm_head"])
            if ragged:
                return [logits[a:b] for a, b in zip(cu_host[:-1], cu_host[1:])]
            return logits.view(B, T, cfg.vocab)
        last = h[cu[1:].long() - 1]
        return self._mm(last.contiguous(), w["lm_head"])

    def _mm(self, x, w, out=None, swiglu=False):
        """Prefill projection out = x @ w.T: the tcgen05 prefill GEMM (csrc/sn_pgemm.cu) in bf16
        (swiglu: w in the SwiGLU-interleaved layout, out = silu(gate) * up); torch in the fp32
        numerics mode, which is the reference-precision path, not a fallback."""
        if x.dtype == torch.bfloat16:
            return ops.gemm_prefill(x, w, out, swiglu_h=self.gu_il[1] if swiglu else 0)
        if swiglu:
            ops.swiglu_il(x @ w.t(), out, *self.gu_il)
            return out
        return torch.mm(x, w.t(), out=out) if out is not None else x @ w.t()

    def _tp_sum(self, t):
        """Prefill: sum a row-parallel projection output (fp32 partials) over the TP group."""
        if self.tp > 1:
            from .dist import allreduce_sum_
            assert t.dtype == torch.float32
            allreduce_sum_(t, self.tp_group)

    def _attn_prefill(self, l, kind, h, out, cu, row_seq, row_pos):
        cfg, st, w = self.cfg, self.state[l], self.w["layers"][l]["mixer"]
        Hq, Hkv, D, P = cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim, cfg.page_size
        rows = h.shape[0]
        window = cfg.window if kind == SWA else 0
        bt = self.swa_block_table if kind == SWA else self.fa_block_table
        qkv = self._mm(h, w["qkv_il"])
        q = torch.empty(rows, Hq, D, device=h.device, dtype=h.dtype)
        k = torch.empty(rows, Hkv, D, device=h.device, dtype=h.dtype)
        v = torch.empty_like(k)
        cont = getattr(self, "_append", None)
        if cont is not None:  # the cached prefix the new tokens can see, read before the append
            prefix = self._gather_prefix(st, bt, window, cont[0])
        ops.rope_kv_append(qkv, row_seq, row_pos, self.seq_lens, self.inv_freq, q, k, v, st["k"], st["v"], bt, Hq,
                           Hkv, D, P, window, pair_il=True)
        o = torch.empty(rows, Hq * D, device=h.device, dtype=h.dtype)
        if cont is None:
            ops.attn_prefill(q, k, v, cu, o, Hq, Hkv, D, window, self.scale_attn)
        else:  # keys per sequence: [cached prefix ; new tokens]
            (pk, pv, k0), cu_host = prefix, self._cu_host
            ks, vs, cu_k, q_off = [], [], [0], []
            for b, (a, c) in enumerate(zip(cu_host[:-1], cu_host[1:])):
                n_pre = cont[0][b] - k0[b]
                ks += [pk[b], k[a:c]]
                vs += [pv[b], v[a:c]]
                cu_k.append(cu_k[-1] + n_pre + (c - a))
                q_off.append(n_pre)
            i32 = dict(device=h.device, dtype=torch.int32)
            ops.attn_prefill(q, torch.cat(ks), torch.cat(vs), cu, o, Hq, Hkv, D, window, self.scale_attn,
                             cu_k=torch.tensor(cu_k, **i32), q_off=torch.tensor(q_off, **i32))
        self._mm(o, w["o"], out)

    def _gather_prefix(self, st, bt, window, pos0):
        """K / V of the cached positions [k0, pos0) of each prefilled slot (k0 = 0 for FA, the
        window start for SWA), from the page pool / ring, as contiguous [n, Hkv, D] tensors."""
        P = self.cfg.page_size
        slots = self._slot_idx.tolist() if self._slot_idx is not None else list(range(len(pos0)))
        pk, pv, k0s = [], [], []
        for slot, p0 in zip(slots, pos0):
            k0 = max(0, p0 - window + 1) if window else 0
            pos = torch.arange(k0, p0, device=self.device)
            ring = pos % window if window else pos
            pages = bt[slot][(ring // P).long()].long()
            offs = (ring % P).long()
            pk.append(st["k"][pages, :, offs])
            pv.append(st["v"][pages, :, offs])
            k0s.append(k0)
        return pk, pv, k0s

    def _delta_prefill(self, kind, l, h, out, cu):
        cfg, st, w = self.cfg, self.state[l], self.w["layers"][l]["mixer"]
        rows = h.shape[0]
        dev = h.device
        n_in = w["w_in"].shape[0]
        proj = torch.empty(rows, -(-n_in // 8) * 8, device=dev, dtype=h.dtype)[:, :n_in]  # 16-byte row pitch
        self._mm(h, w["w_in"], proj)
        if kind == GDN:
            Hk, Hv, D = cfg.gdn_k_heads, cfg.gdn_v_heads, cfg.gdn_head_dim
            C = cfg.gdn_conv_channels
            z_off, b_off = C, C + Hv * D
            a_off = b_off + Hv
            f = None
            gate, gate_stride = proj[:, z_off:], proj.stride(0)
        else:
            Hk = Hv = cfg.kda_heads
            D, R = cfg.kda_head_dim, cfg.kda_rank
            C = cfg.kda_conv_channels
            f1_off, g1_off, b_off, a_off = C, C + R, C + 2 * R, 0
            f = self._mm(proj[:, f1_off:f1_off + R], w["f2"])
            gate = self._mm(proj[:, g1_off:g1_off + R], w["g2"]).add_(w["g2_b"])
            gate_stride = gate.stride(0)
        y = torch.empty(rows, C, device=dev, dtype=h.dtype)
        cont = getattr(self, "_append", None)
        hist = None
        if cont is not None:  # inputs before the first new token come from a snapshot of the rings
            sl = self._slot_idx.long() if self._slot_idx is not None else torch.arange(len(cont[0]), device=dev)
            hist = st["conv"][sl].contiguous()
        ops.conv_prefill(proj, proj.stride(0), y, w["conv_w"], st["conv"], cu, self._slot_idx, C, cfg.conv_width,
                         ring_hist=hist, pos0=None if cont is None else cont[1])
        f32 = dict(device=dev, dtype=torch.float32)
        # bf16: chunked WY prefill on tensor cores (GDN scalar gate / KDA per-channel gate);
        # fp32 I/O (1e-4 parity mode): the recurrent scan (same outputs, token-sequential)
        chunked = h.dtype == torch.bfloat16 and getattr(self, "chunked_prefill", True)
        # the chunked passes read q / k as bf16 TMA tiles
        qk_dt = torch.bfloat16 if chunked else torch.float32
        qn = torch.empty(rows, Hk, D, device=dev, dtype=qk_dt)
        kn = torch.empty(rows, Hk, D, device=dev, dtype=qk_dt)
        gexp = torch.empty(rows, Hv, D, **f32) if kind == KDA else torch.empty(rows, Hv, **f32)
        beta = torch.empty(rows, Hv, **f32)
        k_code = 1 if kind == KDA else 0
        glog = (torch.empty(rows, Hv, D, **f32) if kind == KDA else torch.empty(rows, Hv, **f32)) if chunked else None
        ops.delta_prep(k_code, y, proj, b_off, a_off, f, w["A_log"], w["dt_bias"], qn, kn, gexp, beta, Hk, Hv, D,
                       1.0 / math.sqrt(D), cfg.l2_eps, glog=glog)
        o = torch.empty(rows, Hv, D, **f32)
        if chunked:
            self._chunked_delta(kind, qn, kn, y, 2 * Hk * D, glog, beta, o, st["S"], cu, Hk, Hv, D)
        else:
            ops.delta_scan(k_code, qn, kn, y, 2 * Hk * D, gexp, beta, o, st["S"], self._slot_idx, cu, Hk, Hv, D,
                           init_state=cont is not None)
        y_out = torch.empty(rows, Hv * D, device=dev, dtype=h.dtype)
        ops.gated_rmsnorm(o, gate, gate_stride, w["norm_w"], y_out, Hv, D, cfg.mixer_norm_eps, act=k_code)
        self._mm(y_out, w["o"], out)

    def _chunked_delta(self, kind, qn, kn, y, v_off, glog, beta, o, S, cu, Hk, Hv, D, ws_cap=2 << 30):
        """Two-phase chunked prefill over groups of consecutive sequences whose chunk workspace
        fits ws_cap bytes (ragged lengths: the chunk plan follows cu_seqlens)."""
        slot_idx = getattr(self, "_slot_idx", None)
        B = S.shape[0] if slot_idx is None else slot_idx.numel()
        cu_host = getattr(self, "_cu_host", None)
        if cu_host is None or len(cu_host) != B + 1:
            cu_host = [int(x) for x in cu.tolist()]
        lib = ops._lib.load()
        ws_fn = lib.sn_kda_chunk_workspace_bytes if kind == KDA else lib.sn_gdn_chunk_workspace_bytes
        chunks_of = [-(-(b1 - b0) // 64) for b0, b1 in zip(cu_host[:-1], cu_host[1:])]
        b0 = 0
        while b0 < B:
            b1, n = b0, 0
            while b1 < B and (b1 == b0 or ws_fn(n + chunks_of[b1], Hv, D) <= ws_cap):
                n += chunks_of[b1]
                b1 += 1
            r0, r1 = cu_host[b0], cu_host[b1]
            key = (tuple(cu_host[b0:b1 + 1]),)
            if getattr(self, "_chunk_key", None) != key:
                self._chunk_key = key
                self._chunk_plan = ops.chunk_plan([c - r0 for c in cu_host[b0:b1 + 1]], device=qn.device)
            chunks, c0 = self._chunk_plan
            ws = getattr(self, "_chunk_ws", None)
            # states by slot (continuous batching) or, for a full batch, the slice in prompt order
            S_g, sl = (S[b0:b1], None) if slot_idx is None else (S, slot_idx[b0:b1])
            init = getattr(self, "_append", None) is not None  # continuation: start from the live state
            if kind == KDA:
                self._chunk_ws = ops.kda_chunk_prefill2(qn[r0:r1], kn[r0:r1], y[r0:r1], v_off, glog[r0:r1],
                                                        beta[r0:r1], chunks, c0, o[r0:r1], S_g, sl, Hv, D,
                                                        init_state=init, workspace=ws)
            else:
                self._chunk_ws = ops.gdn_chunk_prefill2(qn[r0:r1], kn[r0:r1], y[r0:r1], v_off, glog[r0:r1],
                                                        beta[r0:r1], chunks, c0, o[r0:r1], S_g, sl, Hk, Hv,
                                                        D, init_state=init, workspace=ws)
            b0 = b1

    def _gdn_prefill(self, l, h, out, cu):
        self._delta_prefill(GDN, l, h, out, cu)

    def _kda_prefill(self, l, h, out, cu):
        self._delta_prefill(KDA, l, h, out, cu)

    # ------------------------------------------------------------------ introspection for tests
    def recurrent_state(self, layer):
        """[B, Hv, K, V] view of a GDN/KDA state (stored [B, Hv, V, K])."""
        return self.state[layer]["S"].transpose(-1, -2)


class KernelProbe:
    """Timing events around named kernels.  Created with external=True so that, when the decode
    step is captured into a CUDA graph, the records become graph event nodes on the launching
    stream; after each replay `collect()` returns {name: [ms per launch]}."""

    def __init__(self, fine: bool = False):
        self.pairs = {}
        self._open = {}
        self.fine = fine  # also time norms / GEMMs / elementwise kernels (step breakdown)

    def begin(self, name):
        e = torch.cuda.Event(enable_timing=True, external=True)
        e.record()
        self._open[name] = e

    def end(self, name):
        e = torch.cuda.Event(enable_timing=True, external=True)
        e.record()
        self.pairs.setdefault(name, []).append((self._open.pop(name), e))

    def collect(self):
        return {n: [a.elapsed_time(b) for a, b in ps] for n, ps in self.pairs.items()}
