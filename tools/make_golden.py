"""Generate the committed golden fixtures under tests/golden/.

  placeopt_golden.json  — outputs of the REFERENCE's own placement / cost API
                          (imported from /root/reference/pkg/src in the build
                          container; the GPU box has no /root/reference, so the
                          outputs are frozen here): code<->name codecs, error
                          messages, preset allocations and cost labels, and the
                          reference loader's parse of our ThroughputRecord JSONL.
  fla_pinning.pt        — FLA 0.5.1 naive GDN/KDA recurrences (third-party
                          realisation of R/PAPER.md:1565-1625) on small seeded
                          inputs, frozen so the oracle pinning test also runs
                          where FLA is absent.
  tiny_logits.pt        — oracle logits for BASELINE.json configs 1/2 (tiny
                          supernet, B=1, 512 prefill + 64 decode) at a few
                          positions, plus final recurrent states (fp32 weights).

Run from the repo root:  python tools/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys
import tempfile

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLD = os.path.join(ROOT, "tests", "golden")
REF_SRC = "/root/reference/pkg/src"


def placeopt_golden():
    sys.path.insert(0, REF_SRC)
    import placeopt
    from placeopt import cost as pcost
    from placeopt import placements as pp
    from placeopt.cli import _load_throughput_records

    from paper_2604_19877_b200.placement import PRESETS
    from paper_2604_19877_b200.records import write_records

    cat = pp.DEFAULT_CATALOG
    out = {"placeopt_version_file": os.path.join(REF_SRC, "placeopt/__init__.py"), "codecs": [], "errors": [],
           "presets": {}, "records": None}
    for text in ["ASKG", "AAAA", "GGKKSSAA", "", PRESETS["Reg|Lklhd-10"].layer_string]:
        p = pp.Placement.from_codes(text, cat)
        out["codecs"].append({"codes": text, "assignments": list(p.assignments), "names": p.to_names(cat),
                              "roundtrip": p.to_codes(cat), "counts": list(pp.allocation_of(p).counts)})
    for text in ["ASKX", "a", "AS K"]:
        try:
            pp.Placement.from_codes(text, cat)
        except ValueError as e:
            out["errors"].append({"codes": text, "error": "ValueError", "message": str(e)})
    for bad in [(0, 4), (-1,)]:
        try:
            pp.Placement(tuple(bad), 4)
        except ValueError as e:
            out["errors"].append({"assignments": list(bad), "error": "ValueError", "message": str(e)})
    try:
        cat.index_of("MLA")
    except KeyError as e:
        out["errors"].append({"name": "MLA", "error": "KeyError", "message": str(e)})
    clean = pcost.CostModel((1.0, 0.48, 0.21, 0.14))  # R/PAPER.md:211-214 regression (clean)
    for name, pr in PRESETS.items():
        p = pp.Placement.from_codes(pr.layer_string, cat)
        out["presets"][name] = {
            "layer_string": pr.layer_string,
            "counts": list(pp.allocation_of(p).counts),
            "cost_clean_regression": pcost.allocation_cost(pp.allocation_of(p), clean),
            "placement_cost": pcost.placement_cost(p, clean),
        }
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "r.jsonl")
        rows = [(PRESETS[n].layer_string, 1000.0 + 17 * i) for i, n in enumerate(PRESETS)]
        write_records(path, rows)
        text = open(path).read()
        recs = _load_throughput_records(path, cat)
        out["records"] = {"jsonl": text, "parsed": [[list(r.allocation.counts), r.throughput] for r in recs]}
    out["placeopt_exports"] = sorted(n for n in dir(placeopt) if not n.startswith("_"))
    return out


def fla_pinning():
    from fla.ops.gated_delta_rule.naive import naive_chunk_gated_delta_rule, naive_recurrent_gated_delta_rule
    from fla.ops.kda.naive import naive_chunk_kda, naive_recurrent_kda

    g = torch.Generator().manual_seed(5)
    B, T, H, D = 2, 128, 3, 32
    q = torch.nn.functional.normalize(torch.randn(B, T, H, D, generator=g), dim=-1)
    k = torch.nn.functional.normalize(torch.randn(B, T, H, D, generator=g), dim=-1)
    v = torch.randn(B, T, H, D, generator=g)
    beta = torch.rand(B, T, H, generator=g)
    gs = -torch.rand(B, T, H, generator=g) * 0.5
    gv = -torch.rand(B, T, H, D, generator=g) * 0.5
    h0 = torch.randn(B, H, D, D, generator=g) * 0.1
    o_g, s_g = naive_recurrent_gated_delta_rule(q, k, v, beta, gs, initial_state=h0, output_final_state=True)
    o_gc, s_gc = naive_chunk_gated_delta_rule(q, k, v, gs, beta, initial_state=h0, output_final_state=True)
    o_k, s_k = naive_recurrent_kda(q, k, v, gv, beta, initial_state=h0, output_final_state=True)
    o_kc, s_kc = naive_chunk_kda(q, k, v, gv, beta, initial_state=h0, output_final_state=True)
    return {"inputs": dict(q=q, k=k, v=v, beta=beta, g_scalar=gs, g_vec=gv, h0=h0),
            "gdn": dict(o=o_g, S=s_g, o_chunk=o_gc, S_chunk=s_gc),
            "kda": dict(o=o_k, S=s_k, o_chunk=o_kc, S_chunk=s_kc),
            "source": "fla 0.5.1 naive_recurrent/naive_chunk (3P-FLA/ops/gated_delta_rule/naive.py, "
                      "3P-FLA/ops/kda/naive.py)"}


def tiny_logits():
    from oracle.supernet_oracle import OracleSupernet
    from paper_2604_19877_b200 import TINY
    from paper_2604_19877_b200.placement import GDN, KDA, layer_kinds
    from paper_2604_19877_b200.weights import init_weights

    out = {}
    toks = torch.randint(0, TINY.vocab, (1, 576), generator=torch.Generator().manual_seed(1))
    pick = torch.tensor([0, 1, 127, 128, 255, 511, 512, 540, 575])
    for placement in ("AAAA", "ASKG"):
        kinds = layer_kinds(placement)
        o = OracleSupernet(TINY, kinds, init_weights(TINY, kinds, seed=0), batch=1, max_len=576)
        lg = o.run(toks)
        out[placement] = {"positions": pick, "logits": lg[0, pick].clone(),
                          "states": {l: o.recurrent_state(l).clone() for l, k in enumerate(kinds) if k in (GDN, KDA)}}
    out["tokens"] = toks
    return out


if __name__ == "__main__":
    os.makedirs(GOLD, exist_ok=True)
    with open(os.path.join(GOLD, "placeopt_golden.json"), "w") as f:
        json.dump(placeopt_golden(), f, indent=1, sort_keys=True)
    torch.save(fla_pinning(), os.path.join(GOLD, "fla_pinning.pt"))
    torch.save(tiny_logits(), os.path.join(GOLD, "tiny_logits.pt"))
    print("golden fixtures written to", GOLD)
