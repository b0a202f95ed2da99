"""Placement vocabulary — the drop-in surface of the reference.

Mirrors the public types of the reference's `placeopt.placements`
(R/pkg/src/placeopt/placements.py:19-135): `MixerCatalog`, `DEFAULT_CATALOG`
(FA/SWA/KDA/GDN <-> A/S/K/G), `Placement` (tuple of per-layer type indices
with code-string / name-list codecs) and `Allocation` / `allocation_of`.
Same field names, same argument meaning, same exceptions (ValueError for a bad
code or index, KeyError for an unknown type name), so a `placeopt.Placement`
object can be handed to :class:`~paper_2604_19877_b200.model.Supernet`
unchanged (duck-typed on ``.assignments`` / ``.num_types``).

The runtime's own addition is :func:`layer_kinds`, the immutable per-layer
dispatch table the layer loop and every captured CUDA graph key off
(R/PAPER.md:860-865: "looks up the SupernetConfig to determine which mixer to
run at each layer index ... no global mutable state"), and the Table-4 preset
allocations (R/PAPER.md:962-999) with a pinned layer string for each.
"""
from __future__ import annotations

from dataclasses import dataclass, field

FA, SWA, KDA, GDN = 0, 1, 2, 3
MIXER_NAMES = ("FA", "SWA", "KDA", "GDN")


@dataclass(frozen=True)
class MixerCatalog:
    """Ordered mixer vocabulary; type index i has name names[i] and one-char code short_codes[i]."""

    names: tuple
    short_codes: tuple

    def __post_init__(self) -> None:
        n = len(self.names)
        problems = []
        if n == 0:
            problems.append("catalog needs at least one mixer type")
        elif len(self.short_codes) != n:
            problems.append("one short code per type required")
        elif len(frozenset(self.names)) != n:
            problems.append(f"duplicate type names: {self.names}")
        elif len(frozenset(self.short_codes)) != n:
            problems.append(f"duplicate short codes: {self.short_codes}")
        else:
            bad = [c for c in self.short_codes if len(c) != 1]
            if bad:
                problems.append(f"short codes must be single characters, got {bad[0]!r}")
        if problems:
            raise ValueError(problems[0])

    @property
    def num_types(self) -> int:
        return len(self.names)

    def index_of(self, name: str) -> int:
        for i, known in enumerate(self.names):
            if known == name:
                return i
        raise KeyError(f"unknown mixer type {name!r}; catalog has {self.names}")


DEFAULT_CATALOG = MixerCatalog(names=MIXER_NAMES, short_codes=("A", "S", "K", "G"))


@dataclass(frozen=True)
class Placement:
    """Per-layer mixer choice: assignments[l] is a type index in [0, num_types)."""

    assignments: tuple
    num_types: int

    def __post_init__(self) -> None:
        if self.num_types < 1:
            raise ValueError("num_types must be >= 1")
        out_of_range = [x for x in self.assignments if x < 0 or x >= self.num_types]
        if out_of_range:
            raise ValueError(f"type index {out_of_range[0]} out of range for {self.num_types} types")

    @property
    def num_layers(self) -> int:
        return len(self.assignments)

    def _require(self, catalog: MixerCatalog) -> None:
        if catalog.num_types != self.num_types:
            raise ValueError(f"placement expects {self.num_types} types, catalog has {catalog.num_types}")

    def to_codes(self, catalog: MixerCatalog) -> str:
        self._require(catalog)
        return "".join(map(catalog.short_codes.__getitem__, self.assignments))

    def to_names(self, catalog: MixerCatalog) -> list:
        self._require(catalog)
        return list(map(catalog.names.__getitem__, self.assignments))

    @classmethod
    def from_codes(cls, text: str, catalog: MixerCatalog) -> "Placement":
        index = {code: i for i, code in enumerate(catalog.short_codes)}
        unknown = next((ch for ch in text if ch not in index), None)
        if unknown is not None:
            raise ValueError(f"unknown short code {unknown!r} in {text!r}")
        return cls(tuple(index[ch] for ch in text), catalog.num_types)

    @classmethod
    def from_names(cls, names: list, catalog: MixerCatalog) -> "Placement":
        return cls(tuple(catalog.index_of(n) for n in names), catalog.num_types)


@dataclass(frozen=True)
class Allocation:
    """Layer count per type."""

    counts: tuple

    def __post_init__(self) -> None:
        if not self.counts:
            raise ValueError("allocation needs at least one type")
        if min(self.counts) < 0:
            raise ValueError(f"negative count in allocation {self.counts}")

    @property
    def num_layers(self) -> int:
        return sum(self.counts)

    @property
    def num_types(self) -> int:
        return len(self.counts)


def allocation_of(placement) -> Allocation:
    counts = [0] * placement.num_types
    for x in placement.assignments:
        counts[x] += 1
    return Allocation(tuple(counts))


# ---------------------------------------------------------------- runtime side

def coerce_placement(placement, catalog: MixerCatalog = DEFAULT_CATALOG) -> Placement:
    """Accept a code string ("ASKG..."), a list of names, or any object with
    ``.assignments``/``.num_types`` (our Placement or a ``placeopt.Placement``)."""
    if isinstance(placement, str):
        return Placement.from_codes(placement, catalog)
    if isinstance(placement, (list, tuple)) and placement and isinstance(placement[0], str):
        return Placement.from_names(list(placement), catalog)
    if hasattr(placement, "assignments") and hasattr(placement, "num_types"):
        p = Placement(tuple(int(x) for x in placement.assignments), int(placement.num_types))
        p._require(catalog)
        return p
    raise TypeError(f"cannot interpret {type(placement).__name__} as a placement")


def layer_kinds(placement, catalog: MixerCatalog = DEFAULT_CATALOG) -> tuple:
    """Immutable per-layer dispatch table (FA=0, SWA=1, KDA=2, GDN=3).

    The runtime's kernels are keyed by *name* through the catalog, so a catalog
    with a different order still dispatches each layer to the right mixer."""
    p = coerce_placement(placement, catalog)
    names = p.to_names(catalog)
    return tuple(MIXER_NAMES.index(n) for n in names)


@dataclass(frozen=True)
class Preset:
    name: str
    counts: tuple  # (FA, SWA, KDA, GDN)
    paper_speedup_32k: float | None = None
    source: str = ""
    layer_string: str = field(default="", compare=False)


def spread_layer_string(counts, catalog: MixerCatalog = DEFAULT_CATALOG) -> str:
    """Deterministic placement with a given allocation: at each layer pick the
    type whose prefix count lags its target share the most (ties -> lower
    index).  The paper publishes allocations only (Table 4, R/PAPER.md:962-999;
    SURVEY.md App. A item 8); decode throughput depends on the allocation, not
    the order (R/PAPER.md:219-222), so any member is a valid benchmark layer
    string — this one is pinned so runs are reproducible."""
    L = sum(counts)
    placed = [0] * len(counts)
    out = []
    for layer in range(L):
        lag = [(counts[t] * (layer + 1) / L - placed[t], -t) for t in range(len(counts)) if placed[t] < counts[t]]
        best = -max(lag)[1]
        placed[best] += 1
        out.append(catalog.short_codes[best])
    return "".join(out)


# Table 4 of the paper (R/PAPER.md:962-999), speedups @32k from R/PAPER.md:2219-2225.
_PRESET_TABLE = (
    ("all-FA", (48, 0, 0, 0), 1.0),
    ("Reg|Lklhd-26", (12, 26, 6, 4), 2.85),
    ("Reg|Lklhd-18", (3, 25, 4, 16), 4.76),
    ("Reg|Lklhd-13", (0, 16, 13, 19), 6.9),
    ("Reg|Lklhd-10", (0, 10, 5, 33), 10.69),
    ("Idealized|All-18", (13, 32, 1, 2), 1.99),
    ("Idealized|Lklhd-6", (0, 30, 5, 13), 6.2),
    ("Idealized|All-6", (0, 30, 5, 13), 6.13),
)

PRESETS = {
    name: Preset(name, counts, sp, "R/PAPER.md:962-999", spread_layer_string(counts))
    for name, counts, sp in _PRESET_TABLE
}

FASTEST_PRESET = "Reg|Lklhd-10"


def preset_placement(name: str) -> Placement:
    return Placement.from_codes(PRESETS[name].layer_string, DEFAULT_CATALOG)
