"""Multi-GPU partitioning of the mixer step.

Two modes, one process per GPU (torch.distributed, NCCL over NVLink for the
collectives):

* Batch sharding (configs 3/4): requests are independent, so rank r simply
  decodes its own slice of the request batch with a full replica of the
  placement; there is no data-path collective.  `shard_batch` is the plan.

* Head-parallel tensor parallelism (config 5: one long sequence): every mixer is
  split by heads, Megatron-style — the fused in-projections column-parallel (each
  rank gets the rows of its heads, in the same fused layout, so the unchanged
  decode/prefill kernels run with local head counts), the out-projection
  row-parallel (each rank gets the input columns of its heads) followed by ONE
  all-reduce of the [tokens, d] partial output per mixer (R/PAPER.md trains with
  TP-8, :386-388; the north star's "one NCCL all-reduce over NVLink after the
  output projection").  The FFN is split the same way (gate/up rows, down
  columns, one all-reduce).  Per rank at Apriel / TP-8: FA/SWA 4 q + 1 kv head,
  GDN 1 key head + its 4 value heads, KDA 4 heads; KDA's first low-rank factors
  (d -> R) are replicated, the second factors and the output gate bias split by
  head.

Everything here is pure tensor slicing / integer arithmetic, so the plan is
testable on CPU with the gloo backend (tests/test_dist_cpu.py).
"""
from __future__ import annotations

from dataclasses import replace

import torch

from .config import SupernetConfig
from .placement import FA, GDN, KDA, SWA


# ---------------------------------------------------------------- batch sharding
def shard_batch(global_batch: int, world_size: int, rank: int) -> tuple[int, int]:
    """(start, count) of rank's slice; the first global_batch % world ranks get one extra."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise ValueError(f"bad rank {rank} for world size {world_size}")
    base, extra = divmod(global_batch, world_size)
    count = base + (1 if rank < extra else 0)
    start = rank * base + min(rank, extra)
    return start, count


# ---------------------------------------------------------------- head parallel
def tp_config(cfg: SupernetConfig, world: int) -> SupernetConfig:
    """The per-rank config: every head count divided by `world` (and the FFN width)."""
    need = {"n_q_heads": cfg.n_q_heads, "n_kv_heads": cfg.n_kv_heads, "gdn_k_heads": cfg.gdn_k_heads,
            "gdn_v_heads": cfg.gdn_v_heads, "kda_heads": cfg.kda_heads, "ffn": cfg.ffn}
    bad = [k for k, v in need.items() if v % world]
    if bad:
        raise ValueError(f"{cfg.name}: {bad} not divisible by tensor-parallel size {world}")
    return replace(cfg, name=f"{cfg.name}/tp{world}", **{k: v // world for k, v in need.items()})


def _rows(t, start, count):
    return t[start:start + count]


def shard_mixer(cfg: SupernetConfig, kind: int, w: dict, world: int, rank: int) -> dict:
    """Slice one layer's mixer weights (the fused layouts of weights.py) for `rank`."""
    d = cfg.hidden
    if kind in (FA, SWA):
        D, Hq, Hkv = cfg.head_dim, cfg.n_q_heads, cfg.n_kv_heads
        hq, hk = Hq // world, Hkv // world
        qkv = w["qkv"]
        q = _rows(qkv, rank * hq * D, hq * D)
        k = _rows(qkv, Hq * D + rank * hk * D, hk * D)
        v = _rows(qkv, (Hq + Hkv) * D + rank * hk * D, hk * D)
        return {"qkv": torch.cat([q, k, v]).contiguous(),
                "o": w["o"][:, rank * hq * D:(rank + 1) * hq * D].contiguous()}
    if kind == GDN:
        D, Hk, Hv = cfg.gdn_head_dim, cfg.gdn_k_heads, cfg.gdn_v_heads
        hk, hv = Hk // world, Hv // world
        wi = w["w_in"]
        C = (2 * Hk + Hv) * D
        parts = [_rows(wi, rank * hk * D, hk * D),                       # q
                 _rows(wi, Hk * D + rank * hk * D, hk * D),              # k
                 _rows(wi, 2 * Hk * D + rank * hv * D, hv * D),          # v
                 _rows(wi, C + rank * hv * D, hv * D),                   # z
                 _rows(wi, C + Hv * D + rank * hv, hv),                  # b
                 _rows(wi, C + Hv * D + Hv + rank * hv, hv)]             # a
        cw = w["conv_w"]
        conv = torch.cat([_rows(cw, rank * hk * D, hk * D), _rows(cw, Hk * D + rank * hk * D, hk * D),
                          _rows(cw, 2 * Hk * D + rank * hv * D, hv * D)])
        return {"w_in": torch.cat(parts).contiguous(), "conv_w": conv.contiguous(),
                "A_log": w["A_log"][rank * hv:(rank + 1) * hv].contiguous(),
                "dt_bias": w["dt_bias"][rank * hv:(rank + 1) * hv].contiguous(),
                "norm_w": w["norm_w"], "o": w["o"][:, rank * hv * D:(rank + 1) * hv * D].contiguous()}
    if kind == KDA:
        D, H, R = cfg.kda_head_dim, cfg.kda_heads, cfg.kda_rank
        h = H // world
        HD = H * D
        wi = w["w_in"]
        parts = [_rows(wi, i * HD + rank * h * D, h * D) for i in range(3)]    # q, k, v
        parts += [_rows(wi, 3 * HD, R), _rows(wi, 3 * HD + R, R)]               # f1, g1 (replicated)
        parts += [_rows(wi, 3 * HD + 2 * R + rank * h, h)]                      # b
        cw = w["conv_w"]
        conv = torch.cat([_rows(cw, i * HD + rank * h * D, h * D) for i in range(3)])
        sl = slice(rank * h * D, (rank + 1) * h * D)
        return {"w_in": torch.cat(parts).contiguous(), "conv_w": conv.contiguous(),
                "f2": w["f2"][sl].contiguous(), "g2": w["g2"][sl].contiguous(), "g2_b": w["g2_b"][sl].contiguous(),
                "A_log": w["A_log"][rank * h:(rank + 1) * h].contiguous(), "dt_bias": w["dt_bias"][sl].contiguous(),
                "norm_w": w["norm_w"], "o": w["o"][:, rank * h * D:(rank + 1) * h * D].contiguous()}
    raise ValueError(kind)


def shard_ffn(cfg: SupernetConfig, layer: dict, world: int, rank: int) -> dict:
    """Column-parallel gate/up (keeping the [gate | up] layout), row-parallel down."""
    F = cfg.ffn
    f = F // world
    gu = layer["ffn_gu"]
    out = dict(layer)
    out["ffn_gu"] = torch.cat([_rows(gu, rank * f, f), _rows(gu, F + rank * f, f)]).contiguous()
    out["ffn_down"] = layer["ffn_down"][:, rank * f:(rank + 1) * f].contiguous()
    return out


def shard_weights(cfg: SupernetConfig, kinds, weights: dict, world: int, rank: int) -> dict:
    """Per-rank weight structure for head-parallel TP (embedding, norms, LM head replicated)."""
    out = {k: v for k, v in weights.items() if k != "layers"}
    out["layers"] = []
    for l, kind in enumerate(kinds):
        lw = shard_ffn(cfg, weights["layers"][l], world, rank)
        lw["mixer"] = shard_mixer(cfg, kind, weights["layers"][l]["mixer"], world, rank)
        out["layers"].append(lw)
    return out


def allreduce_sum_(t, group=None):
    """In-place sum over the tensor-parallel group (NCCL on GPUs, gloo in CPU tests)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


# ---------------------------------------------------------------- peer-memory all-reduce
class SymmetricSlabs:
    """One fp32 buffer per rank, mapped into every peer of the group through CUDA IPC
    (torch's CUDA-tensor sharing: cudaIpcGetMemHandle / cudaIpcOpenMemHandle, P2P over
    NVLink), for the fused all-reduce + residual + RMSNorm of the head-parallel decode
    (csrc/sn_tp.cu).  Layout: [64-word header: word 0 = arrival counter]
    [parity 0: nsplit_max x rows x dim][parity 1: same].  Collective: every rank of `group`
    must construct it (the handles travel through group.all_gather_object)."""

    HEADER = 64

    def __init__(self, rows: int, dim: int, group=None, nsplit_max: int = 8, device="cuda"):
        import torch.distributed as tdist
        from torch.multiprocessing.reductions import reduce_tensor
        self.world = tdist.get_world_size(group)
        self.rank = tdist.get_rank(group)
        self.rows, self.dim, self.nsplit_max = rows, dim, nsplit_max
        self.region = nsplit_max * rows * dim
        self.buf = torch.zeros(self.HEADER + 2 * self.region, device=device, dtype=torch.float32)
        torch.cuda.synchronize()
        shared = [None] * self.world
        tdist.all_gather_object(shared, reduce_tensor(self.buf), group=group)
        self.peers = []
        for r, (rebuild, args) in enumerate(shared):
            self.peers.append(self.buf if r == self.rank else rebuild(*args))
        base = [p.data_ptr() for p in self.peers]
        self.counters = torch.tensor(base, dtype=torch.int64, device=device)
        self.slab_ptrs = [torch.tensor([b + 4 * (self.HEADER + q * self.region) for b in base], dtype=torch.int64,
                                       device=device) for q in (0, 1)]
        tdist.barrier(group)

    def local_slabs(self, parity: int, nsplit: int = None) -> torch.Tensor:
        """This rank's [nsplit_max, rows, dim] slab view of one parity region."""
        off = self.HEADER + parity * self.region
        return self.buf[off: off + self.region].view(self.nsplit_max, self.rows, self.dim)

    def counter_ptr(self) -> int:
        return self.buf.data_ptr()
