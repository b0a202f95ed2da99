"""Head-parallel TP end to end with two real processes on one GPU: each rank builds the
sharded Supernet (dist.shard_weights, local head counts) and runs the real kernels; the
row-parallel partials meet in torch.distributed all-reduces (gloo here — only one GPU is
available; the same calls run over NCCL on a multi-GPU node).  Rank 0's prefill logits and
decode logits must match the unsharded single-process model.  The decode all-reduces run
through CUDA-IPC peer memory (sn_tp.cu), which two processes on one GPU exercise for real."""
import os
import socket
import tempfile

import pytest
import torch
import torch.multiprocessing as mp

from paper_2604_19877_b200 import TINY

CFG = TINY.scaled(name="tiny-tp2", n_kv_heads=2, gdn_k_heads=2)
PLACEMENT, B, T, STEPS = "ASKG", 2, 80, 4


def _tokens():
    return torch.randint(0, CFG.vocab, (B, T + STEPS), generator=torch.Generator().manual_seed(2))


def _run(model, toks, graph=False):
    outs = [model.prefill(toks[:, :T], return_all=True).float().cpu()]
    if graph:
        from paper_2604_19877_b200.graphs import DecodeGraph
        g = DecodeGraph(model, preserve_state=True)
        for t in range(T, T + STEPS):
            model.step_tokens.copy_(toks[:, t].to(torch.int32))
            g.replay()
            outs.append(model.logits.clone().float().cpu()[:, None])
        torch.cuda.synchronize()
    else:
        for t in range(T, T + STEPS):
            outs.append(model.decode(toks[:, t]).float().cpu()[:, None])
    return torch.cat(outs, 1)


def _worker(rank, world, port, path, graph=False, nccl_path=False):
    import torch.distributed as dist
    from paper_2604_19877_b200.model import Supernet
    from paper_2604_19877_b200.placement import layer_kinds
    from paper_2604_19877_b200.weights import init_weights
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    w = init_weights(CFG, layer_kinds(PLACEMENT), seed=0)
    model = Supernet(CFG, PLACEMENT, batch=B, max_len=T + STEPS, dtype=torch.bfloat16, weights=w,
                     tp_group=dist.group.WORLD, tp_transport="nccl" if nccl_path else "p2p")
    out = _run(model, _tokens(), graph=graph)
    if rank == 0:
        torch.save(out, path)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("graph,nccl_path", [(False, False), (True, False), (False, True)])
def test_tp2_two_processes_match_unsharded(graph, nccl_path):
    """Decode all-reduces through peer memory fused with the norm (default; eager and in a
    CUDA graph), or through torch.distributed (tp_transport="nccl")."""
    from paper_2604_19877_b200.model import Supernet
    from paper_2604_19877_b200.placement import layer_kinds
    from paper_2604_19877_b200.weights import init_weights
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "tp.pt")
        mp.spawn(_worker, args=(2, port, path, graph, nccl_path), nprocs=2, join=True)
        tp_out = torch.load(path)
    ref_model = Supernet(CFG, PLACEMENT, batch=B, max_len=T + STEPS, dtype=torch.bfloat16,
                         weights=init_weights(CFG, layer_kinds(PLACEMENT), seed=0))
    ref = _run(ref_model, _tokens())
    err = ((tp_out - ref).abs().max() / ref.abs().max()).item()
    assert err < 2e-2, err
