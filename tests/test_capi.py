"""The C-ABI library loads without a GPU and exports every symbol include/dchag.h declares."""
import ctypes
import os
import re

from paper_2506_21411_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "dchag.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const char\*|int)\s+(dchag_\w+)\(", hdr, re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("dchag_gemm_bf16", "dchag_l0_logits", "dchag_l0_node", "dchag_combine",
              "dchag_unfold", "dchag_tile_weights", "dchag_version", "dchag_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for s in declared_symbols():
        assert hasattr(lib, s), s
        assert s in _lib.SIGNATURES or s in _lib.STRING_FNS, f"{s} not bound in _lib"
    assert lib.dchag_version().decode().startswith("dchag-b200")


def test_shape_errors_raise_without_launch():
    lib = _lib.load()
    rc = lib.dchag_gemm_bf16(None, 1, 1, 100, 64, 0, 0, 64, None, 64, 0, 64, None, 0, None, 0,
                             0, 1, None, 0, 0, 0, 0, None, 0, 0, 0, None)
    assert rc == 1 and b"gemm" in lib.dchag_last_error()
