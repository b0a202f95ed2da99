"""Host side of §8f items 2-3 on CPU: the trace log-likelihood math, the evaluator's
line-protocol validation (it fails before any GPU work, as the reference's
SubprocessEvaluator expects), and the supernet store handing out exactly the tensors a
standalone engine would draw."""
import math
import os
import subprocess
import sys

import pytest
import torch

from paper_2604_19877_b200 import TINY
from paper_2604_19877_b200.evaluator import loglik_from_logits, parse_placements, synthetic_traces
from paper_2604_19877_b200.placement import layer_kinds
from paper_2604_19877_b200.weights import init_weights

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SRC = "/root/reference/pkg/src"


def test_loglik_from_logits_matches_definition():
    g = torch.Generator().manual_seed(0)
    logits = torch.randn(3, 7, 11, generator=g)
    toks = torch.randint(0, 11, (3, 7), generator=g)
    ll = loglik_from_logits(logits, toks)
    for b in range(3):
        ref = sum(math.log(torch.softmax(logits[b, t], -1)[toks[b, t + 1]].item()) for t in range(6)) / 6
        assert abs(ll[b].item() - ref) < 1e-5
    # a uniform model scores -log(V) per token
    assert torch.allclose(loglik_from_logits(torch.zeros(2, 5, 11), toks[:2, :5]).float(),
                          torch.full((2,), -math.log(11.0)), atol=1e-6)
    # completion-only scoring (R/PAPER.md:917-921): the first 4 tokens are prompt
    llc = loglik_from_logits(logits, toks, prompt_len=4)
    for b in range(3):
        ref = sum(math.log(torch.softmax(logits[b, t], -1)[toks[b, t + 1]].item()) for t in range(3, 6)) / 3
        assert abs(llc[b].item() - ref) < 1e-5
    with pytest.raises(ValueError):
        loglik_from_logits(logits, toks, prompt_len=7)


def test_parse_placements_validates_every_line():
    assert parse_placements(["ASKG", "", " GGGG "], 4) == ["ASKG", "GGGG"]
    with pytest.raises(ValueError, match="line 2"):
        parse_placements(["ASKG", "AXKG"], 4)
    with pytest.raises(ValueError, match="3 layers"):
        parse_placements(["ASK"], 4)


def test_synthetic_traces_are_seeded():
    a, b = synthetic_traces(2, 9, 50, 3), synthetic_traces(2, 9, 50, 3)
    assert torch.equal(a, b) and a.max() < 50


def _run_evaluator(stdin, *args):
    return subprocess.run([sys.executable, "-m", "paper_2604_19877_b200.evaluator", "--config", "tiny", *args],
                          input=stdin, capture_output=True, text=True, cwd=ROOT)


def test_evaluator_rejects_bad_codes_before_gpu_work():
    p = _run_evaluator("ASKG\nAZKG\n")
    assert p.returncode == 2 and "line 2" in p.stderr and p.stdout == ""


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference sources not present")
def test_reference_subprocess_evaluator_sees_our_failure():
    """The reference's own adapter (acquisition.py:312-340) turns our non-zero exit into EvaluatorError."""
    sys.path.insert(0, REF_SRC)
    try:
        from placeopt.acquisition import EvaluatorError, SubprocessEvaluator
        from placeopt.placements import DEFAULT_CATALOG, Placement
    finally:
        sys.path.remove(REF_SRC)
    ev = SubprocessEvaluator([sys.executable, "-m", "paper_2604_19877_b200.evaluator", "--config", "tiny",
                              "--trace-len", "8"], DEFAULT_CATALOG)
    bad = Placement.from_codes("ASKGA", DEFAULT_CATALOG)  # 5 layers: the tiny supernet has 4
    cwd = os.getcwd()
    os.chdir(ROOT)
    try:
        with pytest.raises(EvaluatorError, match="exited with 2"):
            ev.evaluate([bad])
    finally:
        os.chdir(cwd)


def test_store_hands_out_the_standalone_tensors():
    from paper_2604_19877_b200.serving import SupernetStore
    store = SupernetStore(TINY, seed=0, device="cpu", dtype=torch.float32)
    for placement in ("ASKG", "GGKA"):
        w = store.weights(placement)
        ref = init_weights(TINY, layer_kinds(placement), seed=0)
        assert torch.equal(w["embed"], ref["embed"]) and torch.equal(w["lm_head"], ref["lm_head"])
        for lw, rw in zip(w["layers"], ref["layers"]):
            assert torch.equal(lw["ffn_gu"], rw["ffn_gu"])
            for k in rw["mixer"]:
                assert torch.equal(lw["mixer"][k], rw["mixer"][k]), k
    # trunk tensors are shared, not copied, between placements
    assert store.weights("ASKG")["layers"][0]["ffn_gu"] is store.weights("GGKA")["layers"][0]["ffn_gu"]
    with pytest.raises(ValueError, match="layers"):
        store.weights("ASK")


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference sources not present")
def test_speculative_trace_schema_feeds_reference_estimator():
    """Our JSONL rows construct the reference's TraceTokenLogProbs and estimate_acceptance
    (speculative.py:62-94) accepts them."""
    sys.path.insert(0, REF_SRC)
    try:
        from placeopt.speculative import TraceTokenLogProbs, estimate_acceptance
    finally:
        sys.path.remove(REF_SRC)
    rows = [{"prompt_id": "prompt-0", "log_q": [-1.0] * 16, "log_p": [-1.0] * 16},
            {"prompt_id": "prompt-1", "log_q": [-2.0] * 16, "log_p": [-1.0] * 16}]
    est = estimate_acceptance([TraceTokenLogProbs(r["prompt_id"], tuple(r["log_q"]), tuple(r["log_p"])) for r in rows],
                              gamma=8)
    assert est.n_steps == 4 and 0 < est.acceptance_rate <= 1
