"""§8f items 2-3 on the GPU: the trace log-likelihood evaluator (the reference's subprocess
line protocol) against the CPU oracle, and per-request placement routing over one resident
supernet — a request routed inside a mixed batch decodes exactly what its placement decodes
alone."""
import os
import subprocess
import sys

import pytest
import torch

from oracle.supernet_oracle import OracleSupernet
from paper_2604_19877_b200 import TINY
from paper_2604_19877_b200.evaluator import loglik_from_logits, synthetic_traces
from paper_2604_19877_b200.placement import layer_kinds
from paper_2604_19877_b200.weights import cast_weights, init_weights

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_evaluator_line_protocol_matches_oracle_loglik():
    placements = ["ASKG", "AAAA", "GGKS"]
    N, T = 2, 96
    p = subprocess.run([sys.executable, "-m", "paper_2604_19877_b200.evaluator", "--config", "tiny", "--num-traces",
                        str(N), "--trace-len", str(T), "--batch", "2", "--init-device", "cpu"], input="\n".join(placements) + "\n",
                       capture_output=True, text=True, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    scores = [float(x) for x in p.stdout.split()]
    assert len(scores) == len(placements)
    traces = synthetic_traces(N, T, TINY.vocab, 1)
    for code, got in zip(placements, scores):
        kinds = layer_kinds(code)
        w = cast_weights(init_weights(TINY, kinds, seed=0), "cpu", torch.bfloat16)
        logits = OracleSupernet(TINY, kinds, w, batch=N, max_len=T).run(traces)
        ref = float(loglik_from_logits(logits, traces).mean())
        assert abs(got - ref) < 5e-3, (code, got, ref)
    assert len(set(scores)) == len(scores)  # placements are distinguishable


@pytest.mark.gpu
def test_router_matches_standalone_placements():
    from paper_2604_19877_b200.serving import PlacementRouter, SupernetStore
    store = SupernetStore(TINY, seed=0, init_device="cpu")
    g = torch.Generator().manual_seed(5)
    prompts = [torch.randint(0, TINY.vocab, (40,), generator=g) for _ in range(5)]
    reqs = [("ASKG", prompts[0]), ("GGGG", prompts[1]), ("ASKG", prompts[2]), ("AAAA", prompts[3]),
            ("GGGG", prompts[4])]
    router = PlacementRouter(store, max_len=64)
    mixed = router.generate(reqs, max_new_tokens=12)
    # the same requests one placement at a time, on fresh routers (engines rebuilt)
    for code in ("ASKG", "GGGG", "AAAA"):
        idx = [i for i, (c, _) in enumerate(reqs) if c == code]
        alone = PlacementRouter(store, max_len=64).generate([reqs[i] for i in idx], max_new_tokens=12)
        for j, i in enumerate(idx):
            assert torch.equal(mixed[i], alone[j]), (code, i)
    # engines are cached per (placement, batch) and reused
    m1, _ = router.engine("ASKG", 2)
    m2, _ = router.engine("ASKG", 2)
    assert m1 is m2
    # the mixers of every placement share one trunk: resident bytes well under 3 full copies
    full = sum(t.numel() * t.element_size() for t in [store.trunk["embed"], store.trunk["lm_head"]])
    assert store.resident_bytes() < 3 * full + 3 * 10**8


@pytest.mark.gpu
def test_speculative_traces_match_oracle_logprobs():
    from paper_2604_19877_b200.serving import SupernetStore
    from paper_2604_19877_b200.speculative import acceptance_traces
    store = SupernetStore(TINY, seed=0, init_device="cpu")  # the oracle's (CPU-drawn) weights
    prompts = torch.randint(0, TINY.vocab, (2, 24), generator=torch.Generator().manual_seed(3))
    rows = acceptance_traces(store, "GGGG", "AAAA", prompts, completion_len=16)
    assert len(rows) == 2 and all(len(r["log_q"]) == len(r["log_p"]) == 16 for r in rows)
    # the completion is the target's greedy continuation: recompute both log-prob sets on the oracle
    from paper_2604_19877_b200.serving import PlacementRouter
    gen = PlacementRouter(store, max_len=40).generate([("AAAA", prompts[b]) for b in range(2)], 16)
    seqs = torch.cat([prompts, torch.stack(gen).long()], 1)
    for key, code in (("log_p", "AAAA"), ("log_q", "GGGG")):
        kinds = layer_kinds(code)
        w = cast_weights(init_weights(TINY, kinds, seed=0), "cpu", torch.bfloat16)
        logits = OracleSupernet(TINY, kinds, w, batch=2, max_len=40).run(seqs)
        lp = torch.log_softmax(logits[:, 23:-1].float(), -1).gather(-1, seqs[:, 24:, None])[..., 0]
        got = torch.tensor([r[key] for r in rows])
        assert (got - lp).abs().max() < 5e-2, key
    # draft == target: every ratio is 1, so every drafted token is accepted
    same = acceptance_traces(store, "AAAA", "AAAA", prompts, completion_len=8)
    assert all(r["log_q"] == r["log_p"] for r in same)


@pytest.mark.gpu
@pytest.mark.parametrize("target,draft", [("AAAA", "GGGG"), ("AKGA", "GGGG")])
def test_speculative_decoding_is_lossless(target, draft):
    """Self-speculative decoding (draft proposals verified by one append prefill of the target)
    emits exactly the target's own greedy decode (fp32 parity mode, so decode and prefill
    arithmetic agree to 1e-4 and argmax ties cannot flip)."""
    from paper_2604_19877_b200.model import Supernet
    from paper_2604_19877_b200.serving import SupernetStore
    from paper_2604_19877_b200.speculative import speculative_generate
    store = SupernetStore(TINY, seed=0, dtype=torch.float32, init_device="cpu")
    prompt = torch.randint(0, TINY.vocab, (50,), generator=torch.Generator().manual_seed(8))
    n = 24
    spec, accepted = speculative_generate(store, draft, target, prompt, n, gamma=4)
    ref_model = Supernet(TINY, target, batch=1, max_len=50 + n + 8, dtype=torch.float32,
                         weights=store.weights(target))
    t = int(torch.argmax(ref_model.prefill(prompt[None]).float(), dim=-1)[0])
    ref = []
    for _ in range(n):
        ref.append(t)
        t = int(torch.argmax(ref_model.decode(torch.tensor([t], dtype=torch.int32)).float(), dim=-1)[0])
    assert spec.tolist() == ref
    assert len(accepted) >= 1 and all(0 <= a <= 4 for a in accepted)
    # the same draft as target accepts everything
    same, acc_same = speculative_generate(store, target, target, prompt, 12, gamma=4)
    assert all(a == 4 for a in acc_same[:-1])
