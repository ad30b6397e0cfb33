"""ctypes binding of the collm C ABI (``include/collm.h``).

This is the only place the Python host touches native code.  It loads the in-tree
``libcollm.so`` (built by :mod:`paper_2604_16400_b200.build`) and fails loudly when it is missing:
there is no CPU fallback for the product path.  Status codes are mapped to the reference's error
classes (``ConfigurationError`` / ``InvariantViolation``, /root/reference/pkg/src/coserve/domain.py:15-20).
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from .domain import ConfigurationError, InvariantViolation

LIB_PATH = Path(__file__).resolve().parent / "libcollm.so"

COLLM_OK, COLLM_EINVAL, COLLM_EINTERNAL, COLLM_ECUDA, COLLM_EUNSUPPORTED = range(5)
MODE_STORE_GRAD, MODE_ADAMW, MODE_COPY_ONLY = 0, 1, 2

_P = C.c_void_p
_I = C.c_int
_LL = C.c_longlong
_F = C.c_float
_SZ = C.c_size_t
_IP = C.POINTER(C.c_int32)
_FP = C.POINTER(C.c_float)

class ReduceGroup(C.Structure):
    """Mirror of ``collm_reduce_group`` (include/collm.h)."""

    _fields_ = [("U", _P), ("V", _P), ("grad", _P), ("master", _P), ("m", _P), ("v", _P),
                ("out_same", _P), ("out_trans", _P), ("ldu", _I), ("ldv", _I), ("u_off", _I),
                ("P", _I), ("v_off", _I), ("Q", _I), ("ldc", _I), ("ld_trans", _I),
                ("c_row_off", _I), ("c_col_off", _I), ("t_row_off", _I), ("t_col_off", _I),
                ("V2", _P)]


_RGP = C.POINTER(ReduceGroup)

# name -> (restype, argtypes); mirrors include/collm.h one to one (tests check the exports).
SIGNATURES: dict[str, tuple] = {
    "collm_version": (_I, []),
    "collm_last_error": (C.c_char_p, []),
    "collm_device_info": (_I, [_I, _IP, _IP, _IP]),
    "collm_preload": (_I, []),
    "collm_plan_segments": (_I, [_IP, _IP, _I, _I, _IP, _IP, _I, _IP, _IP, _I, _IP]),
    "collm_expand_segments": (_I, [_P, _P, _I, _I, _P, _P, _P, _P, _P]),
    "collm_lora_shrink": (_I, [_P, _I, _P, _LL, _I, _P, _I, _P, _IP, _I, _P, _P, _P, _I, _P, _P,
                               _P, _P, _P, _P]),
    "collm_set_rank_sms": (_I, [_I]),
    "collm_get_rank_sms": (_I, []),
    "collm_set_flash_impl": (_I, [_I]),
    "collm_get_flash_impl": (_I, []),
    "collm_set_reduce_impl": (_I, [_I]),
    "collm_get_reduce_impl": (_I, []),
    "collm_plan_shrink_windows": (_I, [_IP, _I, _I, _I, _IP, _I, _IP, _IP]),
    "collm_shrink_tc_workspace_bytes": (_SZ, [_I, _I]),
    "collm_lora_shrink_tc": (_I, [_P, _I, _I, _P, _LL, _I, _I, _P, _P, _I, _I, _P, _P, _IP, _I,
                                  _P, _P, _P, _I, _P, _P, _P, _P, _SZ, _P]),
    "collm_flash_attention_fwd": (_I, [_P, _I, _P, _I, _P, _I, _P, _I, _P, _I, _I, _I, _I, _P, _P,
                                       _F, _I, _P]),
    "collm_flash_attention_bwd": (_I, [_P, _I, _P, _I, _P, _I, _P, _I, _P, _I, _P, _P, _P, _I, _P,
                                       _I, _P, _I, _I, _I, _I, _I, _P, _P, _F, _I, _P]),
    "collm_cross_entropy": (_I, [_P, _I, _I, _I, _P, _P, _P, _P, _P, _I, _F, _P]),
    "collm_attention_workspace_bytes": (_SZ, [_I, _I, _I, _I]),
    "collm_paged_attention": (_I, [_P, _I, _I, _I, _I, _I, _P, _P, _I, _P, _I, _P, _P, _I, _F,
                                   _P, _I, _P, _SZ, _P]),
    "collm_gemm_workspace_bytes": (_SZ, [_I]),
    "collm_set_gemm_lean": (_I, [_I]),
    "collm_gemm_lora": (_I, [_P, _I, _P, _I, _P, _I, _I, _I, _I, _P, _I, _I, _P, _I, _I, _P, _P,
                             _I, _I, _I, _IP, _IP, _I, _P, _SZ, _P, _P, _I, _P]),
    "collm_gemm_lora_ex": (_I, [_P, _I, _P, _I, _P, _I, _I, _I, _I, _P, _I, _I, _P, _I, _I, _P,
                                _P, _I, _I, _I, _IP, _IP, _I, _P, _SZ, _P, _P, _I, _P, _P]),
    "collm_lora_expand_rows": (_I, [_P, _I, _I, _P, _I, _P, _I, _P, _P, _I, _I, _I, _IP, _IP, _P]),
    "collm_reduce_workspace_bytes": (_SZ, [_RGP, _I, _I]),
    "collm_lora_reduce": (_I, [_I, _RGP, _I, _I, _I, _F, _P, _I, _P, _SZ, _P]),
    "collm_lora_apply": (_I, [_RGP, _I, _I, _P, _P]),
}

_lib = None
_lock = threading.Lock()


class CollmError(RuntimeError):
    """CUDA-level failure inside the collm library (COLLM_ECUDA / COLLM_EUNSUPPORTED)."""


def load(path: Path | None = None) -> C.CDLL:
    """Load (once) and return the library; raises if it has not been built."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        # COLLM_LIB: an alternative build of the same library (A/B timing tools only)
        p = Path(path) if path else Path(os.environ.get("COLLM_LIB", LIB_PATH))
        if not p.exists():
            raise CollmError(
                f"{p} is missing: build it with `python -m paper_2604_16400_b200.build` "
                "(the co-batched LoRA layer has no CPU fallback)")
        lib = C.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        try:  # force-load the kernels (lazy loading can deadlock the two-stream overlap)
            import torch
            if torch.cuda.is_available():
                lib.collm_preload()
        except ImportError:  # pragma: no cover
            pass
        return lib


def check(status: int, what: str) -> None:
    if status == COLLM_OK:
        return
    msg = f"{what}: {load().collm_last_error().decode(errors='replace')}"
    if status == COLLM_EINVAL:
        raise ConfigurationError(msg)
    if status == COLLM_EINTERNAL:
        raise InvariantViolation(msg)
    raise CollmError(msg)


def call(name: str, *args) -> int:
    """Call a status-returning ABI function and raise on failure."""
    st = getattr(load(), name)(*args)
    check(st, name)
    return st


def int_array(values) -> C.Array:
    vals = [int(v) for v in values]
    return (C.c_int32 * max(1, len(vals)))(*vals)


def float_array(values) -> C.Array:
    vals = [float(v) for v in values]
    return (C.c_float * max(1, len(vals)))(*vals)
