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
import os

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
                 device="cuda", seed: int = 0, weights=None, fa_block_table=None, tp_group=None):
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
        self.w = cast_weights(weights, self.device, dtype)
        del weights  # self.w may alias it; the FFN interleave below must free the original rows
        self.inv_freq = cfg.inv_freq().to(device=self.device, dtype=torch.float32)
        self.scale_attn = attn_scale(cfg)
        self._alloc_state(fa_block_table)
        self._alloc_decode_buffers()
        # head-parallel decode: the row-parallel all-reduces run through peer memory, fused into
        # the next residual add + RMSNorm (csrc/sn_tp.cu); SN_TP_NCCL=1 keeps torch.distributed
        self.sym = None
        if self.tp > 1 and not os.environ.get("SN_TP_NCCL"):
            from .dist import SymmetricSlabs
            self.sym = SymmetricSlabs(batch, cfg.hidden, group=tp_group, device=self.device)
        self.probe = None  # optional KernelProbe: CUDA events around the mixer kernels (bench instrumentation)
        self.force_simt = False
        # bf16 decode projections run on the tcgen05 weight-streaming GEMM (libsn100, batch-as-M
        # UMMA, persistent balanced grid; fp32 split-K slabs are summed by the consuming kernel,
        # the gate/up projection fuses SiLU-mul) or on cuBLAS.  Default from in-step B200 A/B
        # runs (tools/step_time.py): ours for the LM head, the fused FFN gate/up and the FFN
        # down-projection, and from B=16 also the mixer out-projection (split-K slabs into the
        # residual add: B=64 9.844 -> 9.809 ms/step, B=16 7.17 -> 7.09; at B=1-4 cuBLAS is
        # faster); cuBLAS for the mixer in-projections (ours +0.23 ms/step at B=64, the
        # consuming mixer kernels start later).  SN_DECODE_GEMMS=all switches every role to ours.
        tc_ok = dtype == torch.bfloat16 and batch <= 128

        default_roles = "lm_head,ffn_down,ffn_gate_up" + (",out_proj" if batch >= 16 else "")
        sel = os.environ.get("SN_DECODE_GEMMS", default_roles).split(",")
        self.sn_gemm = {r: tc_ok and (r in sel or "all" in sel)
                        for r in ("lm_head", "ffn_down", "ffn_gate_up", "in_proj", "attn_qkv", "out_proj")}
        if tc_ok:  # fp32 split-K slabs of the input-side projections, summed by their consumers
            n_in = max([cfg.attn_qkv_width if k in (FA, SWA) else cfg.gdn_in_width if k == GDN else cfg.kda_in_width
                        for k in self.kinds])
            self.slab_in = torch.empty(8, batch, n_in, device=self.device, dtype=torch.float32)
            self.slab_gu = torch.empty(8, batch, 2 * cfg.ffn, device=self.device, dtype=torch.float32)
        self.gu_mode = os.environ.get("SN_GU_MODE", "swiglu_il")
        self.in_mode = os.environ.get("SN_IN_MODE", "store")
        if self.sn_gemm["ffn_gate_up"] and self.gu_mode == "swiglu_il":
            # fused gate/up + SiLU-mul: gate and up rows interleaved in the GEMM's block height
            # the interleaved copy replaces [gate; up] (no doubled FFN weights in HBM); prefill
            # de-interleaves its GEMM output (deinterleave_swiglu)
            ffn = self.cfg.ffn
            hb = ops.gemm_swiglu_block(batch, ffn, self.cfg.hidden)
            self.gu_il = (ffn, hb)
            for lw in self.w["layers"]:
                if "ffn_gu_il" in lw:  # prebuilt and shared (serving.SupernetStore)
                    if lw["ffn_gu_il"].shape[0] != -(-ffn // hb) * 2 * hb:
                        raise ValueError("prebuilt SwiGLU-interleaved FFN weights do not match this batch's block")
                else:
                    lw["ffn_gu_il"] = ops.interleave_swiglu(lw.pop("ffn_gu"), hb)
        else:
            self.gu_il = None
            if any("ffn_gu" not in lw for lw in self.w["layers"]):
                raise ValueError("this engine needs the [gate; up] FFN weights (ffn_gu)")

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
        # fp32 K-split partial slabs of the residual-updating projections (o-proj, FFN down),
        # summed into the residual by the next add_rmsnorm
        self.slab_mix = e(8, B, cfg.hidden, d=torch.float32)
        self.slab_ffn = e(8, B, cfg.hidden, d=torch.float32)
        kinds = set(self.kinds)
        self.dec = {}
        if kinds & {FA, SWA}:
            Hq, Hkv, D = cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim
            self.dec["qkv"] = e(B, cfg.attn_qkv_width)
            self.dec["q"] = e(B, Hq, D)
            self.dec["attn"] = e(B, Hq * D)
            self.dec["counters"] = torch.zeros(B * Hkv, device=dev, dtype=torch.int32)
            self.attn_split = {}
            for kind, max_keys in ((FA, self.max_len), (SWA, cfg.window)):
                if kind in kinds:
                    sp, ms = choose_split(_ceil(max_keys, cfg.page_size), B * Hkv,
                                          cap=int(os.environ.get("SN_SPLIT_CAP", 64)),
                                          floor=int(os.environ.get("SN_SPLIT_FLOOR", 4)),
                                          per_sm=int(os.environ["SN_SPLIT_PER_SM"]) if "SN_SPLIT_PER_SM" in os.environ
                                          else None)
                    self.attn_split[kind] = (sp, ms)
            ms_max = max(ms for _, ms in self.attn_split.values())
            nbytes = ops.attn_decode_workspace_bytes(B, Hq, Hkv, D, ms_max)
            self.dec["ws"] = torch.empty(max(nbytes // 4, 1), device=dev, dtype=torch.float32)
            self.ws_max_splits = ms_max
        if GDN in kinds:
            self.dec["gdn_proj"] = e(B, cfg.gdn_in_width)
            self.dec["gdn_out"] = e(B, cfg.gdn_value_dim)
        if KDA in kinds:
            self.dec["kda_proj"] = e(B, cfg.kda_in_width)
            self.dec["kda_out"] = e(B, cfg.kda_dim)
            self.dec["kda_fg"] = e(2, B, cfg.kda_dim)
            # stacked second low-rank factors [2][R][H*D] for the batched f/gate GEMM
            for l, k in enumerate(self.kinds):
                if k == KDA:
                    mw = self.w["layers"][l]["mixer"]
                    mw["fg2T"] = torch.stack([mw["f2"].t(), mw["g2"].t()]).contiguous()

    # ------------------------------------------------------------------ decode
    def _attn_decode(self, l, kind, h, out):
        cfg, st, w, d = self.cfg, self.state[l], self.w["layers"][l]["mixer"], self.dec
        Hq, Hkv, D, P = cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim, cfg.page_size
        window = cfg.window if kind == SWA else 0
        bt = self.swa_block_table if kind == SWA else self.fa_block_table
        qkv, ns = self._gemm_in(h, w["qkv"], d["qkv"], attn=True)
        self._probe_begin("rope_kv_append", fine=True)
        ops.rope_kv_append(qkv, None, self.positions, self.seq_lens, self.inv_freq, d["q"], None, None,
                           st["k"], st["v"], bt, Hq, Hkv, D, P, window, nsplit=ns)
        self._probe_end("rope_kv_append", fine=True)
        sp, _ = self.attn_split[kind]
        name = "swa_decode" if kind == SWA else "fa_decode"
        self._probe_begin(name)
        ops.attn_decode(d["q"], st["k"], st["v"], bt, self.seq_lens, d["attn"], d["ws"], d["counters"], Hq, Hkv, D,
                        P, window, sp, self.ws_max_splits, self.scale_attn, force_simt=self.force_simt)
        self._probe_end(name)
        return self._gemm_residual(d["attn"], w["o"], self.slab_mix, out, "out_proj")

    def _gdn_decode(self, l, h, out):
        cfg, st, w, d = self.cfg, self.state[l], self.w["layers"][l]["mixer"], self.dec
        D = cfg.gdn_head_dim
        proj, ns = self._gemm_in(h, w["w_in"], d["gdn_proj"])
        self._probe_begin("gdn_decode")
        ops.gdn_decode(proj, st["conv"], w["conv_w"], st["S"], None, self.positions, w["A_log"], w["dt_bias"],
                       w["norm_w"], d["gdn_out"], cfg.gdn_k_heads, cfg.gdn_v_heads, D, cfg.conv_width,
                       1.0 / math.sqrt(D), cfg.l2_eps, cfg.mixer_norm_eps, nsplit=ns)
        self._probe_end("gdn_decode")
        return self._gemm_residual(d["gdn_out"], w["o"], self.slab_mix, out, "out_proj")

    def _kda_decode(self, l, h, out):
        cfg, st, w, d = self.cfg, self.state[l], self.w["layers"][l]["mixer"], self.dec
        D = cfg.kda_head_dim
        proj, ns = self._gemm_in(h, w["w_in"], d["kda_proj"])
        fg = None
        if ns == 0:  # low-rank gate second factors as one batched GEMM (1 MB of weights, read once)
            HD, R = cfg.kda_dim, cfg.kda_rank
            f1g1 = proj[:, 3 * HD:3 * HD + 2 * R].view(self.B, 2, R).transpose(0, 1)
            fg = d["kda_fg"]
            torch.bmm(f1g1, w["fg2T"], out=fg)
        self._probe_begin("kda_decode")
        ops.kda_decode(proj, st["conv"], w["conv_w"], st["S"], None, self.positions, w["A_log"],
                       w["dt_bias"], w["f2"], w["g2"], w["g2_b"], w["norm_w"], d["kda_out"], cfg.kda_heads, D,
                       cfg.kda_rank, cfg.conv_width, 1.0 / math.sqrt(D), cfg.l2_eps, cfg.mixer_norm_eps, nsplit=ns,
                       fg=fg)
        self._probe_end("kda_decode")
        return self._gemm_residual(d["kda_out"], w["o"], self.slab_mix, out, "out_proj")

    def _probe_begin(self, name, fine=False):
        if self.probe is not None and (self.probe.fine or not fine):
            self.probe.begin(name)

    def _probe_end(self, name, fine=False):
        if self.probe is not None and (self.probe.fine or not fine):
            self.probe.end(name)

    def _gemm_in(self, x, w, out_bf16, attn=False):
        """Input-side projection: (tensor, nsplit) for the consuming kernel — bf16 (tcgen05 GEMM
        or cuBLAS), or fp32 split-K slabs of the tcgen05 GEMM summed on load by the consumer.
        Role "in_proj" covers the delta-rule mixers, "attn_qkv" the attention projection (6144
        rows: too few for a balanced unsplit weight stream, cuBLAS by default)."""
        self._probe_begin("gemm_in_proj", fine=True)
        role = "attn_qkv" if attn else "in_proj"
        if self.sn_gemm[role] and self.in_mode == "store":
            ops.gemm_decode(x, w, out_bf16, "store")
            res = (out_bf16, 0)
        elif self.sn_gemm[role]:
            slab = self._slab_view(self.slab_in, w.shape[0])
            res = (slab, ops.gemm_decode(x, w, slab, "partial"))
        else:
            torch.mm(x, w.t(), out=out_bf16)
            res = (out_bf16, 0)
        self._probe_end("gemm_in_proj", fine=True)
        return res

    def _slab_view(self, buf, n):
        """Contiguous [8, B, n] view at the start of a slab buffer (slab stride B*n)."""
        return buf.view(-1)[: 8 * self.B * n].view(8, self.B, n)

    def _gemm_store(self, x, w, out, role):
        self._probe_begin("gemm_" + role, fine=True)
        if self.sn_gemm[role]:
            ops.gemm_decode(x, w, out, "store")
        else:
            torch.mm(x, w.t(), out=out)
        self._probe_end("gemm_" + role, fine=True)

    def _gemm_residual(self, x, w, slab, out_bf16, role):
        """Projection whose result is added to the residual stream.  Returns the pending
        update (delta, partials, nsplit) that the next add_rmsnorm applies."""
        if self.sym is not None:  # row-parallel partial straight into this rank's symmetric slabs
            parity = 0 if role == "out_proj" else 1
            slabs = self.sym.local_slabs(parity)
            if self.dtype == torch.bfloat16:
                ns = ops.gemm_decode(x, w, slabs, "partial")
            else:
                torch.mm(x, w.t(), out=slabs[0])
                ns = 1
            ops.tp_arrive(self.sym.counter_ptr())
            return ("tp", parity, ns)
        if self.tp > 1:  # row-parallel: fp32 partial of this rank, summed over the TP group
            from .dist import allreduce_sum_
            buf = slab[0]
            if self.dtype == torch.bfloat16:
                buf.zero_()
                ops.gemm_decode(x, w, buf, "resid")
            else:
                torch.mm(x, w.t(), out=buf)
            allreduce_sum_(buf, self.tp_group)
            return (None, slab, 1)
        self._probe_begin("gemm_" + role, fine=True)
        if self.sn_gemm[role]:
            ns = ops.gemm_decode(x, w, slab, "partial")
            self._probe_end("gemm_" + role, fine=True)
            return (None, slab, ns)
        torch.mm(x, w.t(), out=out_bf16)
        self._probe_end("gemm_" + role, fine=True)
        return (out_bf16, None, 0)

    def _norm(self, pending, weight):
        delta, part, ns = pending
        if isinstance(delta, str):  # ("tp", parity, nsplit): peer-memory all-reduce fused with the norm
            sym = self.sym
            ops.tp_allreduce_add_rmsnorm(sym.slab_ptrs[part], sym.counters, sym.world, sym.rank, ns, self.residual,
                                         weight, self.h, self.cfg.norm_eps)
            return
        self._probe_begin("add_rmsnorm", fine=True)
        ops.add_rmsnorm(delta, self.residual, weight, self.h, self.cfg.norm_eps, partials=part, nsplit=ns)
        self._probe_end("add_rmsnorm", fine=True)

    def decode_body(self):
        """One decode step on the current stream: step_tokens -> logits, next_tokens.
        Graph-capturable: every size/position it needs is read from device buffers."""
        cfg, w = self.cfg, self.w
        self._probe_begin("embed", fine=True)
        ops.embed(self.step_tokens, w["embed"], self.residual, self.seq_lens, self.positions)
        self._probe_end("embed", fine=True)
        pending = (None, None, 0)
        for l, kind in enumerate(self.kinds):
            lw = w["layers"][l]
            self._norm(pending, lw["norm1"])
            if kind == GDN:
                pending = self._gdn_decode(l, self.h, self.mix_out)
            elif kind == KDA:
                pending = self._kda_decode(l, self.h, self.mix_out)
            else:
                pending = self._attn_decode(l, kind, self.h, self.mix_out)
            self._norm(pending, lw["norm2"])
            self._probe_begin("gemm_ffn_gate_up", fine=True)
            if self.sn_gemm["ffn_gate_up"] and self.gu_mode == "swiglu_il":
                ops.gemm_decode(self.h, lw["ffn_gu_il"], self.act, "swiglu_il")
                self._probe_end("gemm_ffn_gate_up", fine=True)
            else:
                if self.sn_gemm["ffn_gate_up"]:
                    gu, ns = self.slab_gu, ops.gemm_decode(self.h, lw["ffn_gu"], self.slab_gu, "partial")
                else:
                    torch.mm(self.h, lw["ffn_gu"].t(), out=self.gu)
                    gu, ns = self.gu, 0
                self._probe_end("gemm_ffn_gate_up", fine=True)
                self._probe_begin("silu_mul", fine=True)
                ops.silu_mul(gu, self.act, nsplit=ns)
                self._probe_end("silu_mul", fine=True)
            pending = self._gemm_residual(self.act, lw["ffn_down"], self.slab_ffn, self.ffn_out, "ffn_down")
        self._norm(pending, w["final_norm"])
        self._gemm_store(self.h, w["lm_head"], self.logits, "lm_head")
        self._probe_begin("argmax", fine=True)
        ops.argmax(self.logits, self.next_tokens)
        self._probe_end("argmax", fine=True)

    def kernels_per_step(self) -> dict:
        """Launch census of one decode step: {"sn": libsn100 kernels, "cublas": library GEMMs}."""
        g = self.sn_gemm
        sn = 3                                 # embed, final norm, argmax
        lib = 0
        sn, lib = (sn + 1, lib) if g["lm_head"] else (sn, lib + 1)
        for kind in self.kinds:
            sn += 2                            # two add_rmsnorm
            sn += 2 if kind in (FA, SWA) else 1    # rope+attention | fused delta-rule decode
            for role in ("attn_qkv" if kind in (FA, SWA) else "in_proj", "out_proj", "ffn_down", "ffn_gate_up"):
                sn, lib = (sn + 1, lib) if g[role] else (sn, lib + 1)
            if kind == KDA and not g["in_proj"]:
                lib += 1                       # low-rank gate second factors (batched GEMM)
            if not (g["ffn_gate_up"] and self.gu_mode == "swiglu_il"):
                sn += 1                        # silu_mul (fused into the gate/up GEMM otherwise)
        return {"sn": sn, "cublas": lib}

    @torch.no_grad()
    def decode(self, tokens):
        """Eager decode step.  tokens: [B] ints (any device) -> logits [B, V] (device buffer)."""
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
        h, mix, ffn_o = e(rows, cfg.hidden), e(rows, cfg.hidden), e(rows, cfg.hidden)
        ops.embed(flat, w["embed"], resid)
        delta = None
        for l, kind in enumerate(self.kinds):
            lw = w["layers"][l]
            ops.add_rmsnorm(delta, resid, lw["norm1"], h, cfg.norm_eps)
            if kind in (FA, SWA):
                self._attn_prefill(l, kind, h, mix, cu, row_seq, row_pos)
            elif kind == GDN:
                self._gdn_prefill(l, h, mix, cu)
            else:
                self._kda_prefill(l, h, mix, cu)
            self._tp_sum(mix)
            ops.add_rmsnorm(mix, resid, lw["norm2"], h, cfg.norm_eps)
            act = e(rows, cfg.ffn)
            if self.gu_il is not None:
                ops.swiglu_il(h @ lw["ffn_gu_il"].t(), act, *self.gu_il)
            else:
                ops.silu_mul(h @ lw["ffn_gu"].t(), act)
            torch.mm(act, lw["ffn_down"].t(), out=ffn_o)
            self._tp_sum(ffn_o)
            delta = ffn_o
        ops.add_rmsnorm(delta, resid, w["final_norm"], h, cfg.norm_eps)
        if return_all:
            logits = h @ w["lm_head"].t()
            if ragged:
                return [logits[a:b] for a, b in zip(cu_host[:-1], cu_host[1:])]
            return logits.view(B, T, cfg.vocab)
        last = h[cu[1:].long() - 1]
        return last @ w["lm_head"].t()

    def _tp_sum(self, t):
        """Prefill: sum a row-parallel projection output over the TP group (in fp32)."""
        if self.tp > 1:
            from .dist import allreduce_sum_
            if t.dtype == torch.float32:
                allreduce_sum_(t, self.tp_group)
            else:
                t32 = t.float()
                allreduce_sum_(t32, self.tp_group)
                t.copy_(t32)

    def _attn_prefill(self, l, kind, h, out, cu, row_seq, row_pos):
        cfg, st, w = self.cfg, self.state[l], self.w["layers"][l]["mixer"]
        Hq, Hkv, D, P = cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim, cfg.page_size
        rows = h.shape[0]
        window = cfg.window if kind == SWA else 0
        bt = self.swa_block_table if kind == SWA else self.fa_block_table
        qkv = h @ w["qkv"].t()
        q = torch.empty(rows, Hq, D, device=h.device, dtype=h.dtype)
        k = torch.empty(rows, Hkv, D, device=h.device, dtype=h.dtype)
        v = torch.empty_like(k)
        cont = getattr(self, "_append", None)
        if cont is not None:  # the cached prefix the new tokens can see, read before the append
            prefix = self._gather_prefix(st, bt, window, cont[0])
        ops.rope_kv_append(qkv, row_seq, row_pos, self.seq_lens, self.inv_freq, q, k, v, st["k"], st["v"], bt, Hq,
                           Hkv, D, P, window)
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
        torch.mm(o, w["o"].t(), out=out)

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
        proj = h @ w["w_in"].t()
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
            f = (proj[:, f1_off:f1_off + R] @ w["f2"].t()).contiguous()
            gate = (proj[:, g1_off:g1_off + R] @ w["g2"].t() + w["g2_b"]).contiguous()
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
        qn, kn = torch.empty(rows, Hk, D, **f32), torch.empty(rows, Hk, D, **f32)
        gexp = torch.empty(rows, Hv, D, **f32) if kind == KDA else torch.empty(rows, Hv, **f32)
        beta = torch.empty(rows, Hv, **f32)
        k_code = 1 if kind == KDA else 0
        # bf16: chunked WY prefill on tensor cores (GDN scalar gate / KDA per-channel gate);
        # fp32 I/O (1e-4 parity mode): the recurrent scan (same outputs, token-sequential)
        chunked = h.dtype == torch.bfloat16 and getattr(self, "chunked_prefill", True)
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
        torch.mm(y_out, w["o"].t(), out=out)

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
