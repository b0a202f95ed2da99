"""Multi-process (gloo, world_size 2, CPU) checks of the multi-GPU plans:

* head-parallel TP: each rank runs the oracle on its `dist.shard_weights` slice with the
  per-rank `dist.tp_config`, one all-reduce after every mixer out-projection and FFN
  down-projection; the result must equal the single-device oracle.
* batch sharding: ranks decode disjoint request slices with no collective; gathering
  their logits reproduces the full batch (to CPU-BLAS rounding, which depends on the
  matrix height; on the GPU the per-row arithmetic is batch-size independent).
"""
import os

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_19877_b200 import TINY

CFG = TINY.scaled(name="tiny-tp", n_kv_heads=2, gdn_k_heads=2)
PLACEMENT = "AGKS"
T = 24


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.set_num_threads(1)


def _tp_worker(rank, world, port, q):
    from oracle.supernet_oracle import OracleSupernet
    from paper_2604_19877_b200.dist import shard_weights, tp_config
    from paper_2604_19877_b200.placement import layer_kinds
    from paper_2604_19877_b200.weights import init_weights
    _init(rank, world, port)
    kinds = layer_kinds(PLACEMENT)
    full = init_weights(CFG, kinds, seed=7)
    toks = torch.randint(0, CFG.vocab, (2, T), generator=torch.Generator().manual_seed(11))
    local = OracleSupernet(tp_config(CFG, world), kinds, shard_weights(CFG, kinds, full, world, rank), batch=2,
                           max_len=T)

    def allreduce(t):
        t = t.contiguous()
        dist.all_reduce(t)
        return t
    local.reduce = allreduce
    got = local.run(toks)
    if rank == 0:
        ref = OracleSupernet(CFG, kinds, full, batch=2, max_len=T).run(toks)
        q.put(((got - ref).abs().max() / ref.abs().max()).item())
    dist.barrier()
    dist.destroy_process_group()


def _batch_worker(rank, world, port, q):
    from oracle.supernet_oracle import OracleSupernet
    from paper_2604_19877_b200.dist import shard_batch
    from paper_2604_19877_b200.placement import layer_kinds
    from paper_2604_19877_b200.weights import init_weights
    _init(rank, world, port)
    kinds = layer_kinds(PLACEMENT)
    w = init_weights(CFG, kinds, seed=7)
    toks = torch.randint(0, CFG.vocab, (5, 12), generator=torch.Generator().manual_seed(3))
    start, count = shard_batch(5, world, rank)
    mine = OracleSupernet(CFG, kinds, w, batch=count, max_len=12).run(toks[start:start + count])
    parts = [None] * world
    dist.all_gather_object(parts, mine)
    if rank == 0:
        full = OracleSupernet(CFG, kinds, w, batch=5, max_len=12).run(toks)
        q.put(((torch.cat(parts) - full).abs().max() / full.abs().max()).item())
    dist.destroy_process_group()


def _run(fn, port):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=fn, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_head_parallel_tp2_matches_single_device():
    err = _run(_tp_worker, 29517)
    assert err < 1e-5, err


def test_batch_sharding_matches_full_batch():
    assert _run(_batch_worker, 29518) < 1e-5


def test_tp_config_rejects_indivisible():
    from paper_2604_19877_b200.dist import tp_config
    with pytest.raises(ValueError):
        tp_config(TINY, 2)  # one kv head cannot be split two ways
