"""The C-ABI library loads (no GPU needed) and exports every symbol include/sn_abi.h declares,
with the argument counts the ctypes binding uses."""
import os
import re
import subprocess

from paper_2604_19877_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = open(os.path.join(ROOT, "include", "sn_abi.h")).read()


def declared():
    body = re.sub(r"/\*.*?\*/", "", HEADER, flags=re.S)
    out = {}
    for m in re.finditer(r"\b(?:sn_status|size_t|int|const char\*|void)\s+(sn_\w+)\s*\(([^)]*)\)\s*;", body):
        args = m.group(2).strip()
        out[m.group(1)] = 0 if args in ("", "void") else len(args.split(","))
    return out


def test_library_loads_and_exports_all_symbols():
    lib = _lib.load()
    assert lib.sn_abi_version() == _lib.ABI_VERSION
    syms = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (sn_\w+)", syms))
    decl = declared()
    assert len(decl) >= 18
    missing = set(decl) - exported
    assert not missing, f"declared but not exported: {missing}"


def test_ctypes_signatures_match_header():
    decl = declared()
    for name, nargs in decl.items():
        if name in ("sn_last_error",):
            continue
        assert name in _lib.SIGNATURES, f"{name} has no ctypes binding"
        assert len(_lib.SIGNATURES[name]) == nargs, f"{name}: header has {nargs} args"


def test_error_path_without_gpu():
    """Argument validation happens before any CUDA call: a bad call fails cleanly on CPU."""
    lib = _lib.load()
    st = lib.sn_gdn_decode(None, 0, None, None, None, None, None, None, None, None, None, 1, 1, 1, 128, 4,
                           1.0, 1e-6, 1e-5, 1, None)
    assert st == 1 and b"NULL" in lib.sn_last_error()
    st = lib.sn_attn_decode(None, None, None, None, None, None, None, None, 1, 32, 7, 128, 64, 8, 0, 1, 1, 1.0, 1,
                            None)
    assert st == 1


def test_decode_gemm_plans_without_gpu():
    """The decode GEMM plan is host arithmetic (148 SMs assumed without a device): every Apriel
    decode projection keeps >= 96 CTAs streaming; fused modes keep their block constraints."""
    from paper_2604_19877_b200 import APRIEL, ops
    cfg = APRIEL
    for N, K, mode in ((cfg.gdn_in_width, cfg.hidden, "store"), (cfg.hidden, cfg.ffn, "partial"),
                       (cfg.hidden, cfg.gdn_value_dim, "partial"), (cfg.ffn, cfg.hidden, "swiglu_il"),
                       (cfg.attn_qkv_width, cfg.hidden, "attn_in"), (cfg.vocab, cfg.hidden, "store")):
        p = ops.gemm_decode_plan(64, N, K, mode)
        assert 96 <= p["grid"] <= 148 and p["stages"] >= 3, (N, K, p)
        if mode == "swiglu_il":  # 2h rows per block, h a multiple of 16 filling the SMs best
            assert p["br"] == 2 * ops.gemm_swiglu_block(N) and p["br"] % 32 == 0 and p["splits"] == 1
        if mode == "attn_in":
            assert p["br"] % 32 == 0 and p["splits"] == 1
        if mode == "store":
            assert p["splits"] == 1
    assert ops.gemm_swiglu_block(cfg.ffn) == 112  # 14336 / 112 = 128 blocks, one wave on 148 SMs


def test_rope_pair_interleave_is_a_permutation():
    import torch
    from paper_2604_19877_b200 import TINY, ops
    c = TINY
    w = torch.arange(c.attn_qkv_width, dtype=torch.float32)[:, None].repeat(1, 3)
    il = ops.rope_pair_interleave(w, c.n_q_heads, c.n_kv_heads, c.head_dim)
    assert sorted(il[:, 0].tolist()) == w[:, 0].tolist()
    D, half = c.head_dim, c.head_dim // 2
    assert il[0, 0] == 0 and il[1, 0] == half and il[2, 0] == 1 and il[D, 0] == D
    v0 = (c.n_q_heads + c.n_kv_heads) * D
    assert torch.equal(il[v0:], w[v0:])
