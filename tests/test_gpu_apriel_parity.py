"""End-to-end parity at Apriel widths (reduced depth) against the oracle.

The tiny configuration (d=256, head dim 64) never reaches the kernels the benchmark runs:
the tcgen05 attention prefill (head dim 128 only), the decode-GEMM plans of a d=5120 trunk
(split-K slabs, the SwiGLU-interleaved 224-row blocks, the 14336-wide down-projection, the
131072-row LM head), and the delta-rule decode CTAs at 128x128 states in both widths (the
512-thread CTAs of small batches and the 256-thread ones of B=64).  Here every layer has the
Apriel-1.6 shapes (R/PAPER.md:175-182, 1540-1625) and only the depth is cut to 4 layers, one
of each mixer, with the SWA window cut to 256 so a ~300-token prompt wraps the ring.

Flow: a ragged prefill (lengths 300 / 273 / 129 / 64 — ring wrap, chunk boundaries and a
single-chunk prompt, packed in one prefill), then 8 graph-replayed decode steps.  The oracle
(fp32, teacher-forced token by token) runs per group of equal-length prompts.  It runs the same
fp32 torch code as on the CPU, on the GPU with TF32 off, only so that Apriel widths finish in
seconds; it is still the checker, not the product.

Tolerance (north_star): max-abs error / max |ref| <= 2e-2 in bf16, on every prefill
position's logits, every decode step's logits and the final GDN/KDA states.  The oracle sees
the same bf16-rounded weights (cast back to fp32).
"""
import pytest
import torch

from oracle.supernet_oracle import OracleSupernet
from paper_2604_19877_b200 import APRIEL
from paper_2604_19877_b200.placement import GDN, KDA, layer_kinds
from paper_2604_19877_b200.weights import cast_weights, init_weights

TOL = 2e-2
CFG = APRIEL.scaled(num_layers=4, window=256)
LENS = (300, 273, 129, 64)
STEPS = 8


def _rel(a, b):
    return ((a.float() - b.float()).abs().max() / b.float().abs().max().clamp_min(1e-6)).item()


@pytest.fixture(autouse=True)
def _no_tf32():
    old = torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    yield
    torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32 = old


@pytest.mark.gpu
@pytest.mark.parametrize("placement,B,chain", [("SKGA", 64, False), ("AGKS", 64, False), ("SKGA", 1, False),
                                               ("AGKS", 1, False), ("AGKS", 64, True), ("SKGA", 1, True)])
def test_apriel_shapes_ragged_prefill_graph_decode(placement, B, chain):
    """chain=True: the decode step through the fused decode chains (csrc/sn_chain.cu)."""
    from paper_2604_19877_b200.graphs import DecodeGraph
    from paper_2604_19877_b200.model import Supernet

    dev = torch.device("cuda")
    kinds = layer_kinds(placement)
    w = cast_weights(init_weights(CFG, kinds, seed=0, device=dev), dev, torch.bfloat16)
    lens = [LENS[b % len(LENS)] for b in range(B)]
    g = torch.Generator().manual_seed(7)
    seqs = [torch.randint(0, CFG.vocab, (L + STEPS,), generator=g) for L in lens]
    max_len = max(lens) + STEPS

    model = Supernet(CFG, placement, batch=B, max_len=max_len, dtype=torch.bfloat16, weights=w, fused_chain=chain)
    assert model.use_chain == chain
    pre = model.prefill([s[:L] for s, L in zip(seqs, lens)], return_all=True)
    graph = DecodeGraph(model, preserve_state=True)
    dec = []
    for t in range(STEPS):
        model.step_tokens.copy_(torch.tensor([int(s[L + t]) for s, L in zip(seqs, lens)], dtype=torch.int32))
        graph.replay()
        dec.append(model.logits.clone())
    torch.cuda.synchronize()
    assert int(model.err_flag.item()) == 0

    for L in sorted(set(lens)):
        members = [b for b in range(B) if lens[b] == L]
        toks = torch.stack([seqs[b] for b in members])
        oracle = OracleSupernet(CFG, kinds, w, batch=len(members), max_len=L + STEPS, device=dev)
        ref = oracle.run(toks)  # [n, L + STEPS, V]
        for i, b in enumerate(members):
            got = torch.cat([pre[b], torch.stack([d[b] for d in dec])])
            err = _rel(got, ref[i])
            assert err <= TOL, f"{placement} B={B} seq {b} (len {L}): logits rel err {err:.3e}"
        for l, kind in enumerate(kinds):
            if kind in (GDN, KDA):
                got_s = model.recurrent_state(l)[members]
                err = _rel(got_s, oracle.recurrent_state(l))
                assert err <= TOL, f"{placement} B={B} len {L} layer {l}: state rel err {err:.3e}"
        del oracle, ref
