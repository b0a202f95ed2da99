"""The placement vocabulary mirrors the reference's placeopt API bit-exactly.

Golden values in tests/golden/placeopt_golden.json were produced by the REFERENCE
itself (R/pkg/src/placeopt imported in the build container; tools/make_golden.py)."""
import json
import os

import pytest

from paper_2604_19877_b200.placement import (DEFAULT_CATALOG, FASTEST_PRESET, PRESETS, Allocation, MixerCatalog,
                                             Placement, allocation_of, coerce_placement, layer_kinds,
                                             preset_placement, spread_layer_string)

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "placeopt_golden.json")))


def test_catalog_codes():
    assert DEFAULT_CATALOG.names == ("FA", "SWA", "KDA", "GDN")
    assert DEFAULT_CATALOG.short_codes == ("A", "S", "K", "G")
    assert DEFAULT_CATALOG.num_types == 4
    assert [DEFAULT_CATALOG.index_of(n) for n in ("FA", "SWA", "KDA", "GDN")] == [0, 1, 2, 3]


@pytest.mark.parametrize("case", GOLD["codecs"], ids=lambda c: c["codes"] or "<empty>")
def test_codecs_match_reference(case):
    p = Placement.from_codes(case["codes"], DEFAULT_CATALOG)
    assert list(p.assignments) == case["assignments"]
    assert p.to_names(DEFAULT_CATALOG) == case["names"]
    assert p.to_codes(DEFAULT_CATALOG) == case["roundtrip"]
    assert list(allocation_of(p).counts) == case["counts"]
    assert Placement.from_names(case["names"], DEFAULT_CATALOG) == p


@pytest.mark.parametrize("case", GOLD["errors"], ids=lambda c: str(c.get("codes", c.get("assignments", c.get("name")))))
def test_errors_match_reference(case):
    exc = {"ValueError": ValueError, "KeyError": KeyError}[case["error"]]
    with pytest.raises(exc) as info:
        if "codes" in case:
            Placement.from_codes(case["codes"], DEFAULT_CATALOG)
        elif "assignments" in case:
            Placement(tuple(case["assignments"]), 4)
        else:
            DEFAULT_CATALOG.index_of(case["name"])
    msg = str(info.value)
    assert msg == case["message"]


@pytest.mark.parametrize("name", sorted(PRESETS))
def test_presets_match_reference_allocations_and_costs(name):
    g = GOLD["presets"][name]
    pr = PRESETS[name]
    assert pr.layer_string == g["layer_string"]
    assert list(pr.counts) == g["counts"]
    assert list(allocation_of(preset_placement(name)).counts) == g["counts"]
    # the paper's regression cost labels (R/PAPER.md:211-214: 1, 0.48, 0.21, 0.14)
    cost = sum(n * c for n, c in zip(pr.counts, (1.0, 0.48, 0.21, 0.14)))
    assert cost == pytest.approx(g["cost_clean_regression"], abs=1e-9)


def test_fastest_preset_is_reg_lklhd_10():
    assert FASTEST_PRESET == "Reg|Lklhd-10"
    assert PRESETS[FASTEST_PRESET].counts == (0, 10, 5, 33)
    assert sum(n * c for n, c in zip(PRESETS[FASTEST_PRESET].counts, (1, .48, .21, .14))) == pytest.approx(10.47)


def test_layer_kinds_dispatch_table():
    assert layer_kinds("ASKG") == (0, 1, 2, 3)
    assert layer_kinds(["GDN", "FA"]) == (3, 0)
    assert isinstance(layer_kinds("AAAA"), tuple)
    # a catalog in another order still dispatches by name
    cat = MixerCatalog(("GDN", "FA", "SWA", "KDA"), ("g", "a", "s", "k"))
    assert layer_kinds("gask", cat) == (3, 0, 1, 2)


def test_coerce_accepts_placeopt_like_objects():
    class Foreign:  # duck-typed placeopt.Placement
        assignments = (0, 3, 3, 1)
        num_types = 4
    assert coerce_placement(Foreign()).to_codes(DEFAULT_CATALOG) == "AGGS"
    with pytest.raises(TypeError):
        coerce_placement(3.5)
    with pytest.raises(ValueError):
        coerce_placement("ASKX")


def test_spread_layer_string_allocation_exact():
    for counts in [(48, 0, 0, 0), (0, 10, 5, 33), (13, 32, 1, 2), (1, 1, 1, 1)]:
        s = spread_layer_string(counts)
        assert tuple(allocation_of(Placement.from_codes(s, DEFAULT_CATALOG)).counts) == counts


def test_catalog_validation():
    with pytest.raises(ValueError):
        MixerCatalog((), ())
    with pytest.raises(ValueError):
        MixerCatalog(("A", "A"), ("x", "y"))
    with pytest.raises(ValueError):
        MixerCatalog(("A", "B"), ("x", "xy"))
    with pytest.raises(ValueError):
        Allocation((1, -1))
    with pytest.raises(ValueError):
        Placement((0,), 0)


REF_SRC = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="the reference checkout exists only in the build container")
def test_real_placeopt_placement_drives_the_dispatch_table():
    """A real placeopt.Placement (the reference's own type, R/pkg/src/placeopt/placements.py)
    is accepted at the boundary and dispatches every layer like its code string; a reference
    placement over a custom catalog dispatches by mixer name."""
    import sys
    sys.path.insert(0, REF_SRC)
    try:
        from placeopt import placements as pp
    finally:
        sys.path.remove(REF_SRC)
    from paper_2604_19877_b200 import PRESETS
    for text in ["ASKG", "GGKKSSAA", PRESETS["Reg|Lklhd-10"].layer_string]:
        ref = pp.Placement.from_codes(text, pp.DEFAULT_CATALOG)
        assert layer_kinds(ref) == layer_kinds(text)
        assert coerce_placement(ref).to_codes(DEFAULT_CATALOG) == ref.to_codes(pp.DEFAULT_CATALOG)
    ref_alloc = pp.allocation_of(pp.Placement.from_codes(PRESETS["Reg|Lklhd-10"].layer_string, pp.DEFAULT_CATALOG))
    assert tuple(ref_alloc.counts) == PRESETS["Reg|Lklhd-10"].counts
