"""ctypes binding of libsn100.so (include/sn_abi.h).

This is the same binding a reference-side maintainer would add:
plain pointers, ints and floats, a cudaStream_t passed as void*.  The library is
built in-tree (paper_2604_19877_b200/libsn100.so, `make -C paper_2604_19877_b200/csrc`)
and there is no fallback: importing an op without it raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsn100.so")

P = ctypes.c_void_p
I = ctypes.c_int
Fl = ctypes.c_float

# name -> argtypes (restype is int status unless noted)
SIGNATURES = {
    "sn_abi_version": [],
    "sn_embed": [P, P, P, P, P, P, P, I, I, I, I, P],
    "sn_add_rmsnorm": [P, P, I, P, P, P, I, I, Fl, I, P],
    "sn_argmax": [P, I, I, P, P, I, P],
    "sn_swiglu_il": [P, I, P, I, I, I, I, P],
    "sn_rope_kv_append": [P, P, P, P, P, P, P, P, P, P, P, I, I, I, I, I, I, I, I, I, P],
    "sn_attn_decode_workspace_bytes": [I, I, I, I, I],
    "sn_attn_decode": [P, P, P, P, P, P, P, P, I, I, I, I, I, I, I, I, I, Fl, I, P],
    "sn_attn_prefill": [P, P, P, P, P, P, P, I, I, I, I, I, I, I, Fl, I, P],
    "sn_gdn_decode": [P, I, P, P, P, P, P, P, P, P, P, I, I, I, I, I, Fl, Fl, Fl, I, P],
    "sn_kda_decode": [P, I, P, P, P, P, P, P, P, P, P, P, P, I, I, I, I, I, Fl, Fl, Fl, I, P],
    "sn_conv_prefill": [P, I, P, P, P, P, P, P, P, I, I, I, I, I, P],
    "sn_delta_prep": [I, P, P, I, I, I, P, P, P, P, P, P, P, P, I, I, I, I, Fl, Fl, I, I, P],
    "sn_gdn_chunk_workspace_bytes": [I, I, I],
    "sn_gdn_chunk_prefill2": [P, P, P, I, I, I, P, P, P, P, I, P, P, P, P, I, I, I, I, I, I, P],
    "sn_kda_chunk_workspace_bytes": [I, I, I],
    "sn_tp_arrive": [P, P],
    "sn_tp_allreduce_add_rmsnorm": [P, P, I, I, I, P, P, P, I, I, Fl, I, P],
    "sn_kda_chunk_prefill2": [P, P, P, I, I, I, P, P, P, P, I, P, P, P, P, I, I, I, I, I, P],
    "sn_delta_scan": [I, P, P, P, I, I, P, P, P, P, P, P, I, I, I, I, I, I, P],
    "sn_gated_rmsnorm": [P, P, I, P, P, I, I, I, Fl, I, I, P],
    "sn_gemm_swiglu_block": [I],
    "sn_gemm_decode_plan": [I, I, I, I, P],
    "sn_gemm_decode_tune": [I, I, I, I],
    "sn_gemm_decode": [P, I, I, I, P, I, I, P, I, I, P, I, P],
    "sn_gemm_decode_attn_in": [P, I, I, I, P, I, P, P, P, P, P, P, I, I, I, I, I, I, P, P, I, P],
    "sn_decode_chain": [P, I, I, P, P],
    "sn_gemm_prefill": [P, I, I, I, P, I, I, P, I, I, I, P],
    "sn_decode_chain_trace": [P],
}


class ChainPhase(ctypes.Structure):
    """Mirror of include/sn_abi.h sn_chain_phase (field order and types must match)."""
    _fields_ = [
        ("kind", I), ("depends", I),
        ("x", P), ("K", I), ("ldx", I), ("w", P), ("N", I), ("ldw", I), ("out", P), ("ldo", I), ("mode", I),
        ("positions", P), ("inv_freq", P), ("q_out", P), ("k_cache", P), ("v_cache", P), ("block_table", P),
        ("Hq", I), ("Hkv", I), ("D", I), ("page_size", I), ("max_blocks", I), ("window", I), ("err_flag", P),
        ("rope_cs", P),
        ("partials", P), ("nsplit", I), ("residual", P), ("weight", P), ("norm_out", P), ("dim", I), ("eps", Fl),
        ("ss_out", P), ("ss_in", P), ("n_ss", I), ("splits", I),
    ]


SN_CHAIN_GEMM, SN_CHAIN_NORM = 0, 1
RESTYPES = {"sn_gdn_chunk_workspace_bytes": ctypes.c_size_t, "sn_kda_chunk_workspace_bytes": ctypes.c_size_t,
            "sn_attn_decode_workspace_bytes": ctypes.c_size_t,
            "sn_abi_version": ctypes.c_int, "sn_gemm_swiglu_block": ctypes.c_int, "sn_gemm_decode_plan": ctypes.c_int,
            "sn_gemm_decode_tune": None, "sn_decode_chain_trace": None}

SN_F32, SN_BF16 = 0, 1
SN_GEMM_STORE, SN_GEMM_RESID, SN_GEMM_PARTIAL, SN_GEMM_SWIGLU_IL, SN_GEMM_ATTN_IN = 0, 2, 3, 4, 6
ABI_VERSION = 2

_lib = None


class SnError(RuntimeError):
    pass


def load(path: str = LIB_PATH):
    """Load libsn100.so (once) and attach signatures.  Raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"libsn100.so not found at {path}: build it with `make -C paper_2604_19877_b200/csrc` "
            "(there is no CPU fallback for the mixer step)")
    lib = ctypes.CDLL(path)
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = RESTYPES.get(name, ctypes.c_int)
    lib.sn_last_error.argtypes = []
    lib.sn_last_error.restype = ctypes.c_char_p
    if lib.sn_abi_version() != ABI_VERSION:
        raise ImportError(f"libsn100.so ABI {lib.sn_abi_version()} != expected {ABI_VERSION}")
    _lib = lib
    return lib


def call(name: str, *args):
    lib = load()
    st = getattr(lib, name)(*args)
    if st != 0:
        msg = lib.sn_last_error().decode(errors="replace")
        raise SnError(f"{name} failed with status {st}: {msg}")
    return st
