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
    st = lib.sn_gdn_decode(None, 0, 0, None, None, None, None, None, None, None, None, None, 1, 1, 1, 128, 4,
                           1.0, 1e-6, 1e-5, 1, None)
    assert st == 1 and b"NULL" in lib.sn_last_error()
    st = lib.sn_attn_decode(None, None, None, None, None, None, None, None, 1, 32, 7, 128, 64, 8, 0, 1, 1, 1.0, 1,
                            None)
    assert st == 1
