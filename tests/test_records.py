"""Our measured throughput is emitted in the reference's ThroughputRecord JSONL format
(R/SPEC.md:192, parsed by placeopt.cli._load_throughput_records, R/pkg/src/placeopt/cli.py:163-176).
The golden JSONL and its parse were produced with the reference's own loader."""
import json
import os

import pytest

from paper_2604_19877_b200.placement import PRESETS
from paper_2604_19877_b200.records import read_records, throughput_record, write_records

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "placeopt_golden.json")))


def test_jsonl_identical_to_golden(tmp_path):
    rows = [(PRESETS[n].layer_string, 1000.0 + 17 * i) for i, n in enumerate(PRESETS)]
    path = tmp_path / "r.jsonl"
    write_records(str(path), rows)
    assert path.read_text() == GOLD["records"]["jsonl"]
    parsed = read_records(str(path))
    assert [[list(c), t] for c, t in parsed] == GOLD["records"]["parsed"]


def test_record_validation(tmp_path):
    with pytest.raises(ValueError):
        throughput_record("AS", 0.0)
    with pytest.raises(ValueError):
        throughput_record("AS", float("nan"))
    bad = tmp_path / "bad.jsonl"
    bad.write_text('{"counts": {"FA": 1}, "throughput": 3}\n{"counts": {"FA": 2}}\n')
    with pytest.raises(ValueError, match="line 2"):
        read_records(str(bad))
