"""End-to-end parity of the CUDA path against the CPU oracle (BASELINE.json configs 1-2).

Tolerances (north_star): max-abs error / max |ref| <= 1e-4 with fp32 I/O,
<= 2e-2 with bf16 I/O, on logits and recurrent states.  In bf16 mode the oracle
runs on the same bf16-rounded weights (cast back to fp32) so the comparison
isolates the kernels' arithmetic from weight quantisation.
"""
import pytest
import torch

from oracle.supernet_oracle import OracleSupernet
from paper_2604_19877_b200 import TINY
from paper_2604_19877_b200.placement import FA, GDN, KDA, SWA, layer_kinds
from paper_2604_19877_b200.weights import cast_weights, init_weights

TOL = {torch.float32: 1e-4, torch.bfloat16: 2e-2}


def rel_err(a, b):
    a, b = a.detach().float().cpu(), b.detach().float().cpu()
    return ((a - b).abs().max() / b.abs().max().clamp_min(1e-6)).item()


def run_pair(placement, dtype, B, T_prefill, n_decode, cfg=TINY, seed=0, graph=False, force_simt=False, chain=False):
    from paper_2604_19877_b200.model import Supernet
    kinds = layer_kinds(placement)
    w = init_weights(cfg, kinds, seed=seed)
    w = cast_weights(w, "cpu", dtype)  # round once; oracle sees the same values
    g = torch.Generator().manual_seed(1)
    toks = torch.randint(0, cfg.vocab, (B, T_prefill + n_decode), generator=g)
    oracle = OracleSupernet(cfg, kinds, w, batch=B, max_len=T_prefill + n_decode)
    ref = oracle.run(toks)
    model = Supernet(cfg, placement, batch=B, max_len=T_prefill + n_decode, dtype=dtype, weights=w, fused_chain=chain)
    model.force_simt = force_simt
    pre = model.prefill(toks[:, :T_prefill], return_all=True)
    outs = [pre]
    if graph:
        from paper_2604_19877_b200.graphs import DecodeGraph
        dg = DecodeGraph(model, preserve_state=True)
        for t in range(T_prefill, T_prefill + n_decode):
            model.step_tokens.copy_(toks[:, t].to(torch.int32))
            dg.replay()
            outs.append(model.logits.clone()[:, None])
    else:
        for t in range(T_prefill, T_prefill + n_decode):
            outs.append(model.decode(toks[:, t]).clone()[:, None])
    torch.cuda.synchronize()
    got = torch.cat(outs, dim=1)
    return model, oracle, got, ref


def check_states(model, oracle, tol):
    for l, kind in enumerate(model.kinds):
        if kind in (GDN, KDA):
            err = rel_err(model.recurrent_state(l), oracle.recurrent_state(l))
            assert err <= tol, f"layer {l} state rel err {err}"


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("placement", ["AAAA", "ASKG", "GGGG", "KKKK", "SSSS"])
def test_tiny_prefill_decode(placement, dtype):
    model, oracle, got, ref = run_pair(placement, dtype, B=2, T_prefill=200, n_decode=16)
    tol = TOL[dtype]
    assert rel_err(got[:, :200], ref[:, :200]) <= tol
    assert rel_err(got[:, 200:], ref[:, 200:]) <= tol
    check_states(model, oracle, tol)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("placement", ["AAAA", "ASKG"])
def test_baseline_configs_1_2(placement, dtype):
    """BASELINE.json configs 1/2: B=1, 512-token prefill + 64 decode steps (SWA ring wraps: w=128)."""
    model, oracle, got, ref = run_pair(placement, dtype, B=1, T_prefill=512, n_decode=64)
    tol = TOL[dtype]
    assert rel_err(got, ref) <= tol
    check_states(model, oracle, tol)


@pytest.mark.gpu
def test_large_batch_graph_decode():
    """B=96 (> 64: the decode GEMMs switch to the 128-row batch tile, the attention / delta
    kernels get more CTAs than SMs) through prefill and graphed decode."""
    model, oracle, got, ref = run_pair("ASKG", torch.bfloat16, B=96, T_prefill=48, n_decode=6, graph=True)
    assert rel_err(got, ref) <= TOL[torch.bfloat16]
    check_states(model, oracle, TOL[torch.bfloat16])


@pytest.mark.gpu
def test_simt_attention_path_matches_oracle():
    """The CUDA-core decode attention (bf16 cross-check path) is also within tolerance."""
    model, oracle, got, ref = run_pair("ASAS", torch.bfloat16, B=2, T_prefill=150, n_decode=20, force_simt=True)
    assert rel_err(got, ref) <= TOL[torch.bfloat16]


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_graph_replay_equals_eager(dtype):
    """CUDA-graph replay is bit-identical to eager decode (R/PAPER.md:1012-1013 saw graph-mode
    instabilities in third-party kernels; ours must not have any)."""
    _, _, eager, _ = run_pair("ASKG", dtype, B=2, T_prefill=64, n_decode=12)
    _, _, graphed, _ = run_pair("ASKG", dtype, B=2, T_prefill=64, n_decode=12, graph=True)
    assert torch.equal(eager.cpu(), graphed.cpu())


@pytest.mark.gpu
@pytest.mark.parametrize("placement", ["ASKG", "GKSA"])
def test_ragged_prefill_matches_per_sequence_oracle(placement):
    """Prompts of different lengths in one packed prefill (cu_seqlens through every kernel,
    tiles straddling sequences, chunk plans per sequence), then graphed decode: each sequence
    matches the oracle run on that sequence alone."""
    from paper_2604_19877_b200.graphs import DecodeGraph
    from paper_2604_19877_b200.model import Supernet
    kinds = layer_kinds(placement)
    w = cast_weights(init_weights(TINY, kinds, seed=0), "cpu", torch.bfloat16)
    lens, steps = [37, 150, 64], 4
    g = torch.Generator().manual_seed(3)
    seqs = [torch.randint(0, TINY.vocab, (L + steps,), generator=g) for L in lens]
    model = Supernet(TINY, placement, batch=len(lens), max_len=max(lens) + steps, dtype=torch.bfloat16, weights=w)
    pre = model.prefill([s[:L] for s, L in zip(seqs, lens)], return_all=True)
    graph = DecodeGraph(model, preserve_state=True)
    dec = []
    for t in range(steps):
        model.step_tokens.copy_(torch.tensor([int(s[L + t]) for s, L in zip(seqs, lens)], dtype=torch.int32))
        graph.replay()
        dec.append(model.logits.clone().float().cpu())
    torch.cuda.synchronize()
    for b, (s, L) in enumerate(zip(seqs, lens)):
        ref = OracleSupernet(TINY, kinds, w, batch=1, max_len=L + steps).run(s[None])[0]
        got = torch.cat([pre[b].float().cpu(), torch.stack([d[b] for d in dec])])
        assert rel_err(got, ref) <= TOL[torch.bfloat16], (b, rel_err(got, ref))


@pytest.mark.gpu
@pytest.mark.parametrize("placement", ["ASKG", "GKSA"])
def test_continuous_batching_slot_prefill(placement):
    """Prefill into a subset of engine slots while the others keep decoding: slot-indexed KV
    pages / SWA rings / conv tails / recurrent states; every slot matches the oracle run of
    its own token stream."""
    from paper_2604_19877_b200.model import Supernet
    kinds = layer_kinds(placement)
    w = cast_weights(init_weights(TINY, kinds, seed=0), "cpu", torch.bfloat16)
    g = torch.Generator().manual_seed(11)
    lens = {0: 40, 2: 70, 1: 55}
    n1, n2 = 3, 3  # decode steps before / after slot 1 joins
    toks = {s: torch.randint(0, TINY.vocab, (L + n1 + n2,), generator=g) for s, L in lens.items()}
    model = Supernet(TINY, placement, batch=3, max_len=80, dtype=torch.bfloat16, weights=w)
    got = {s: [] for s in lens}
    first = model.prefill([toks[0][:lens[0]], toks[2][:lens[2]]], slots=[0, 2])
    got[0].append(first[0].float().cpu())
    got[2].append(first[1].float().cpu())
    step = {0: lens[0], 2: lens[2], 1: None}

    def decode_all():
        feed = torch.zeros(3, dtype=torch.int32)
        for s in (0, 1, 2):
            if step[s] is not None:
                feed[s] = int(toks[s][step[s]])
        lg = model.decode(feed).float().cpu()
        for s in (0, 1, 2):
            if step[s] is not None:
                got[s].append(lg[s])
                step[s] += 1

    for _ in range(n1):
        decode_all()
    joined = model.prefill([toks[1][:lens[1]]], slots=[1])
    got[1].append(joined[0].float().cpu())
    step[1] = lens[1]
    for _ in range(n2):
        decode_all()
    torch.cuda.synchronize()
    for s, L in lens.items():
        n = len(got[s]) - 1  # decode steps taken by this slot
        ref = OracleSupernet(TINY, kinds, w, batch=1, max_len=L + n).run(toks[s][None, :L + n])[0]
        want = ref[L - 1:L + n]
        assert rel_err(torch.stack(got[s]), want) <= TOL[torch.bfloat16], (s, rel_err(torch.stack(got[s]), want))


@pytest.mark.gpu
@pytest.mark.parametrize("placement", ["ASKG", "GKSA"])
def test_chunked_prompt_append_matches_oracle(placement):
    """A prompt prefilled in pieces (append=True: positions continue, attention reads the
    cached prefix — FA pages and the SWA ring, window 128 smaller than the prompt — conv rings
    and recurrent states carry over) and then decoded matches the oracle on the whole stream."""
    from paper_2604_19877_b200.model import Supernet
    kinds = layer_kinds(placement)
    w = cast_weights(init_weights(TINY, kinds, seed=0), "cpu", torch.bfloat16)
    g = torch.Generator().manual_seed(21)
    total, steps = [230, 150], 3
    pieces = [[64, 100, 66], [1, 129, 20]]
    seqs = [torch.randint(0, TINY.vocab, (T + steps,), generator=g) for T in total]
    model = Supernet(TINY, placement, batch=2, max_len=max(total) + steps, dtype=torch.bfloat16, weights=w)
    got = [[], []]
    for i in range(3):
        a = [sum(p[:i]) for p in pieces]
        chunk = [s[a[b]:a[b] + pieces[b][i]] for b, s in enumerate(seqs)]
        lg = model.prefill(chunk, return_all=True, append=i > 0)
        for b in range(2):
            got[b].append(lg[b].float().cpu())
    for t in range(steps):
        lg = model.decode(torch.tensor([int(s[T + t]) for s, T in zip(seqs, total)], dtype=torch.int32))
        for b in range(2):
            got[b].append(lg[b].float().cpu()[None])
    torch.cuda.synchronize()
    for b, (s, T) in enumerate(zip(seqs, total)):
        ref = OracleSupernet(TINY, kinds, w, batch=1, max_len=T + steps).run(s[None])[0]
        out = torch.cat(got[b])
        assert out.shape[0] == T + steps
        assert rel_err(out, ref) <= TOL[torch.bfloat16], (b, rel_err(out, ref))


@pytest.mark.gpu
@pytest.mark.parametrize("placement", ["ASKG", "GKSA"])
@pytest.mark.parametrize("B", [2, 96])
def test_fused_chain_decode_matches_oracle(placement, B):
    """The fused decode chains (one persistent launch per layer boundary, csrc/sn_chain.cu):
    eager and graphed decode within the bf16 tolerance, graph bit-identical to eager."""
    m1, oracle, eager, ref = run_pair(placement, torch.bfloat16, B=B, T_prefill=70, n_decode=10, chain=True)
    assert m1.use_chain
    assert rel_err(eager, ref) <= TOL[torch.bfloat16]
    check_states(m1, oracle, TOL[torch.bfloat16])
    _, _, graphed, _ = run_pair(placement, torch.bfloat16, B=B, T_prefill=70, n_decode=10, graph=True, chain=True)
    assert torch.equal(eager.cpu(), graphed.cpu())


@pytest.mark.gpu
@pytest.mark.parametrize("placement", ["ASKG", "GKSA"])
def test_idle_slot_does_not_advance(placement):
    """A negative step token marks an idle slot (continuous batching): its length, KV pages /
    ring, conv ring and recurrent state stay untouched, the feedback token stays -1, and when it
    resumes it continues exactly where it stopped (matches the oracle on its own stream)."""
    from paper_2604_19877_b200.graphs import DecodeGraph
    from paper_2604_19877_b200.model import Supernet
    kinds = layer_kinds(placement)
    w = cast_weights(init_weights(TINY, kinds, seed=0), "cpu", torch.bfloat16)
    T, steps, idle = 40, 6, (1, 2, 3)  # slot 1 idles during steps 1..3
    toks = torch.randint(0, TINY.vocab, (3, T + steps), generator=torch.Generator().manual_seed(4))
    model = Supernet(TINY, placement, batch=3, max_len=T + steps, dtype=torch.bfloat16, weights=w)
    model.prefill(toks[:, :T])
    graph = DecodeGraph(model, preserve_state=True)
    got = {0: [], 1: [], 2: []}
    pos = [T, T, T]
    for t in range(steps):
        feed = torch.tensor([int(toks[b, pos[b]]) if not (b == 1 and t in idle) else -1 for b in range(3)],
                            dtype=torch.int32)
        model.step_tokens.copy_(feed)
        graph.replay()
        lg = model.logits.clone().float().cpu()
        nt = model.next_tokens.cpu()
        for b in range(3):
            if b == 1 and t in idle:
                assert int(nt[1]) == -1 and int(model.seq_lens[1]) == pos[1]
                continue
            got[b].append(lg[b])
            pos[b] += 1
    torch.cuda.synchronize()
    assert int(model.err_flag.item()) == 0
    for b in range(3):
        n = len(got[b])
        ref = OracleSupernet(TINY, kinds, w, batch=1, max_len=T + n).run(toks[b:b + 1, :T + n])[0]
        assert rel_err(torch.stack(got[b]), ref[T:T + n]) <= TOL[torch.bfloat16], b
