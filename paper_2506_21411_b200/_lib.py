"""ctypes binding of libdchag.so (the C ABI in include/dchag.h).

The library is built in-tree by `__graft_entry__.build()` / `python -m
paper_2506_21411_b200.build`.  There is no fallback: if the shared object is
missing or a kernel reports an error, the call raises.
"""

from __future__ import annotations

import ctypes
import os

from .config import ConfigError

_HERE = os.path.dirname(os.path.abspath(__file__))
# DCHAG_LIB: an alternative build of the same ABI (A/B timing probes only)
LIB_PATH = os.environ.get("DCHAG_LIB") or os.path.join(_HERE, "libdchag.so")

c_int, c_ll, c_vp = ctypes.c_int, ctypes.c_longlong, ctypes.c_void_p

# name -> argtypes; every function returns int (0 = ok)
SIGNATURES = {
    "dchag_gemm_bf16": [c_vp, c_int, c_int, c_int, c_int, c_ll, c_ll, c_ll, c_vp, c_int, c_ll,
                        c_int, c_vp, c_ll, c_vp, c_ll, c_ll, c_int, c_vp, c_int, c_ll, c_ll,
                        c_ll, c_vp, c_ll, c_ll, c_ll, c_vp],
    "dchag_gemm_nt": [c_vp, c_int, c_ll, c_ll, c_int, c_ll, c_vp, c_int, c_ll, c_ll, c_int,
                      c_int, c_int, c_int, c_vp, c_ll, c_vp, c_int, c_int, c_ll, c_ll, c_vp],
    "dchag_final_vit": [c_vp, c_int, c_int, c_int, c_vp, c_int, c_vp, c_vp, c_vp, c_vp, c_int,
                        c_vp, c_vp, c_vp, c_int, c_vp],
    "dchag_gemm_rowdot": [c_vp, c_int, c_int, c_int, c_int, c_ll, c_ll, c_ll, c_vp, c_int,
                          c_ll, c_vp, c_ll, c_vp, c_ll, c_vp, c_vp],
    "dchag_split3_bf16": [c_vp, c_ll, c_int, c_ll, c_vp, c_ll, c_vp],
    "dchag_l0_p_normalize": [c_vp, c_vp, c_vp, c_vp, c_vp, c_int, c_int, c_int, c_int, c_int,
                             c_vp],
    "dchag_gemm_rowdot_heads": [c_vp, c_int, c_int, c_int, c_int, c_ll, c_ll, c_ll, c_vp, c_int,
                                c_ll, c_vp, c_ll, c_vp, c_ll, c_int, c_vp, c_vp],
    "dchag_gemm_combine": [c_vp, c_int, c_int, c_int, c_int, c_vp, c_ll, c_vp, c_ll, c_vp,
                           c_vp, c_vp, c_int, c_int, c_vp, c_vp],
    "dchag_l0_logits": [c_vp, c_ll, c_ll, c_int, c_int, c_int, c_int, c_int, c_int, c_int,
                        c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp],
    "dchag_l0_node": [c_vp, c_ll, c_ll, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_vp,
                      c_vp, c_vp, c_int, c_vp, c_vp, c_vp, c_int, c_vp, c_int, c_vp, c_vp, c_vp],
    "dchag_combine": [c_int, c_int, c_int, c_int, c_vp, c_vp, c_int, c_vp, c_ll, c_vp, c_ll,
                      c_vp, c_vp, c_vp],
    "dchag_l0_dv": [c_int, c_int, c_int, c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_ll, c_int,
                    c_vp, c_vp, c_vp],
    "dchag_vit_tokens": [c_vp, c_int, c_int, c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_vp],
    "dchag_l0_tgrad": [c_vp, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int,
                       c_vp, c_vp, c_vp, c_vp, c_vp],
    "dchag_child_softmax": [c_vp, c_vp, c_vp, c_int, c_int, c_int, c_vp],
    "dchag_l0_softmax_bwd": [c_int, c_int, c_int, c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_vp,
                             c_vp],
    "dchag_combine_f32": [c_int, c_int, c_int, c_int, c_vp, c_vp, c_int, c_vp, c_ll, c_vp, c_ll,
                          c_vp, c_vp, c_vp],
    "dchag_fullcross_weights": [c_int, c_int, c_int, c_int, c_vp, c_vp, c_int, c_vp, c_ll, c_ll,
                                c_vp, c_ll, c_vp, c_vp, c_int, c_vp, c_vp, c_int, c_vp],
    "dchag_fullcross_bwd": [c_int, c_int, c_int, c_int, c_vp, c_vp, c_int, c_vp, c_ll, c_ll, c_vp,
                            c_vp, c_vp, c_vp, c_vp, c_vp],
    "dchag_combine_weighted": [c_int, c_int, c_int, c_int, c_vp, c_vp, c_int, c_vp, c_ll, c_ll,
                               c_vp, c_vp, c_vp],
    "dchag_combine_strided": [c_int, c_int, c_int, c_int, c_vp, c_vp, c_int, c_vp, c_ll, c_ll,
                              c_vp, c_ll, c_ll, c_int, c_vp, c_vp, c_vp],
    "dchag_combine_bwd": [c_int, c_int, c_int, c_int, c_vp, c_vp, c_int, c_vp, c_ll, c_vp, c_ll,
                          c_vp, c_vp, c_vp, c_vp, c_vp, c_vp],
    "dchag_combine_bwd_packed": [c_int, c_int, c_int, c_int, c_vp, c_vp, c_int, c_vp, c_ll, c_vp,
                                 c_ll, c_vp, c_vp, c_vp, c_ll, c_ll, c_vp, c_vp],
    "dchag_unfold": [c_vp, c_ll, c_ll, c_int, c_int, c_int, c_int, c_int, c_vp, c_vp],
    "dchag_tile_weights": [c_vp, c_int, c_int, c_int, c_vp, c_vp],
    "dchag_l0_tgrad_te": [c_vp, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int,
                          c_vp, c_vp, c_vp, c_vp, c_vp, c_ll, c_int, c_vp],
    "dchag_l0_pack": [c_vp, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int,
                      c_int, c_int, c_ll, c_ll, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                      c_vp, c_vp, c_vp, c_vp, c_vp],
    "dchag_cast_multi": [c_vp, c_int, c_int, c_vp],
    "dchag_query_fold": [c_vp, c_int, c_int, c_int, c_vp, c_vp],
    "dchag_query_fold_bwd": [c_vp, c_int, c_int, c_int, c_vp, c_vp, c_vp],
    "dchag_colsum": [c_vp, c_int, c_ll, c_ll, c_int, c_int, c_int, c_int, c_vp, c_ll, c_ll,
                     c_int, c_int, c_vp, c_vp, c_vp],
    "dchag_rowsum": [c_vp, c_ll, c_int, c_int, c_vp, c_vp],
    "dchag_num_sms": [],
    "dchag_combine_overflow": [c_vp, c_int],
}
STRING_FNS = ("dchag_version", "dchag_last_error")


class ShapeError(ValueError):
    """Unsupported or inconsistent tensor shape (reference tensor.py:29-34)."""


class KernelError(RuntimeError):
    """A CUDA launch failed."""


_lib = None


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the D-CHAG kernels)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = c_int
    for name in STRING_FNS:
        fn = getattr(lib, name)
        fn.argtypes = []
        fn.restype = ctypes.c_char_p
    _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc == 0:
        return
    msg = load().dchag_last_error().decode()
    if rc == 1:
        raise ShapeError(f"{what}: {msg}")
    if rc == 2:
        raise ConfigError(f"{what}: {msg}")
    raise KernelError(f"{what}: {msg}")


# kernel-launch accounting (bench.py reports `gpu_launches`; an optional hook lets the
# bench bracket individual kernels with CUDA events on the launching stream)
LAUNCH_COUNT = {"n": 0}
_HOOK = {"fn": None}
_NON_LAUNCH = ("dchag_num_sms", "dchag_combine_overflow")


def set_launch_hook(fn) -> None:
    """fn(name, phase, work) with phase in {"pre", "post"} around every kernel launch; work
    is the caller's annotation of the launch (site name, algorithmic flops and bytes) or
    None."""
    _HOOK["fn"] = fn


def call(name: str, *args, work: dict | None = None) -> None:
    """Launch one C-ABI entry point; raise on a non-zero status. `work` (optional) annotates
    the launch for measurement: {"site": str, "flops": int, "bytes": int}."""
    hook = _HOOK["fn"]
    if hook is not None:
        hook(name, "pre", work)
    check(getattr(load(), name)(*args), name)
    if name not in _NON_LAUNCH:
        LAUNCH_COUNT["n"] += 1
    if hook is not None:
        hook(name, "post", work)


def ptr(t) -> int:
    """Device pointer of a torch tensor (0 for None)."""
    return 0 if t is None else int(t.data_ptr())


def stream_handle(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
