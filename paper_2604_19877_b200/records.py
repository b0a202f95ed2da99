"""Measured throughput -> the reference's ThroughputRecord JSONL.

The reference consumes throughput only as input records (R/SPEC.md:8, 192):
one JSON object per line, {"counts": {"<type name>": int, ...}, "throughput":
float}, parsed by `placeopt fit-cost` (R/pkg/src/placeopt/cli.py:163-176) and
fit by cost.fit_regression (R/pkg/src/placeopt/cost.py:114-159).  This module
writes exactly that format from our measurements, so `placeopt fit-cost
--records b200.jsonl` refits the paper's additive cost model for B200
(SURVEY.md §8f item 1).
"""
from __future__ import annotations

import json
import math

from .placement import DEFAULT_CATALOG, allocation_of, coerce_placement


def throughput_record(placement, tokens_per_s: float, catalog=DEFAULT_CATALOG) -> dict:
    if not (tokens_per_s > 0 and math.isfinite(tokens_per_s)):
        raise ValueError(f"throughput must be finite and > 0, got {tokens_per_s}")
    p = coerce_placement(placement, catalog)
    counts = allocation_of(p).counts
    return {"counts": {name: int(n) for name, n in zip(catalog.names, counts)}, "throughput": float(tokens_per_s)}


def write_records(path: str, rows) -> None:
    """rows: iterable of (placement, tokens_per_s)."""
    with open(path, "w") as f:
        for placement, tps in rows:
            f.write(json.dumps(throughput_record(placement, tps), sort_keys=True) + "\n")


def read_records(path: str, catalog=DEFAULT_CATALOG):
    """Parse like the reference's loader: returns [(counts tuple, throughput)], ValueError with the
    line number on a malformed line."""
    out = []
    with open(path) as f:
        for lineno, line in enumerate(f, start=1):
            if not line.strip():
                continue
            try:
                row = json.loads(line)
                counts = tuple(int(row["counts"].get(n, 0)) for n in catalog.names)
                tps = float(row["throughput"])
                if not (tps > 0 and math.isfinite(tps)):
                    raise ValueError(f"throughput must be finite and > 0, got {tps}")
            except (KeyError, TypeError, ValueError, json.JSONDecodeError) as exc:
                raise ValueError(f"bad throughput record on line {lineno}: {exc}") from exc
            out.append((counts, tps))
    return out
