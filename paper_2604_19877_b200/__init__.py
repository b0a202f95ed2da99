"""B200-native (sm_100a) runtime for the Super Apriel per-layer mixer step.

Public surface:
  * placement vocabulary mirroring the reference's placeopt API
    (MixerCatalog, DEFAULT_CATALOG, Placement, Allocation, allocation_of, PRESETS)
  * SupernetConfig (TINY, APRIEL), Supernet (prefill/decode), DecodeGraph
  * throughput records in placeopt's ThroughputRecord JSONL format (records.py)

Kernels live in libsn100.so (include/sn_abi.h); importing this package does
not load it, constructing a Supernet does (and fails loudly without it).
"""
from .config import APRIEL, CONFIGS, TINY, SupernetConfig
from .placement import (DEFAULT_CATALOG, FASTEST_PRESET, PRESETS, Allocation, MixerCatalog, Placement,
                        allocation_of, layer_kinds, preset_placement)

__all__ = [
    "APRIEL", "CONFIGS", "TINY", "SupernetConfig", "DEFAULT_CATALOG", "FASTEST_PRESET", "PRESETS", "Allocation",
    "MixerCatalog", "Placement", "allocation_of", "layer_kinds", "preset_placement",
]


def __getattr__(name):
    if name == "Supernet":
        from .model import Supernet
        return Supernet
    if name == "DecodeGraph":
        from .graphs import DecodeGraph
        return DecodeGraph
    raise AttributeError(name)
