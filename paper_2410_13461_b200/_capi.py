"""ctypes binding of the C-ABI library ``lib/libpmpd_b200.so`` (see ``include/pmpd_b200.h``).

The library is the product's only compute path.  Loading fails loudly (no
CPU fallback) when the shared object is missing or no CUDA device is present
at call time.
"""
from __future__ import annotations

import ctypes
import os
import threading

from .errors import ConfigError, ContractViolation, FormatError, InputError, PmpdError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PMPD_LIB") or os.path.join(_HERE, "lib", "libpmpd_b200.so")

OK, ERR_CONFIG, ERR_INPUT, ERR_CONTRACT, ERR_FORMAT, ERR_CUDA = 0, 1, 2, 3, 4, 5
LAYOUT_REF, LAYOUT_KN, LAYOUT_NK = 0, 1, 2
DTYPE_F32, DTYPE_F16, DTYPE_F64 = 0, 1, 2
GEMV_IN_RMSNORM, GEMV_IN_SWIGLU = 1, 2  # pmpd_b200.h PMPD_GEMV_IN_*


class CudaError(PmpdError):
    """A CUDA runtime failure inside the library (no reference counterpart)."""


_ERRORS = {ERR_CONFIG: ConfigError, ERR_INPUT: InputError, ERR_CONTRACT: ContractViolation,
           ERR_FORMAT: FormatError, ERR_CUDA: CudaError}


class QTensorDesc(ctypes.Structure):
    """Mirror of ``pmpd_qtensor``."""
    _fields_ = [("rows", ctypes.c_int32), ("cols", ctypes.c_int32),
                ("group_size", ctypes.c_int32), ("p_max", ctypes.c_int32),
                ("layout", ctypes.c_int32), ("n", ctypes.c_int32), ("k", ctypes.c_int32),
                ("n_tiles", ctypes.c_int32), ("k_tiles", ctypes.c_int32), ("groups", ctypes.c_int32),
                ("plane_bytes", ctypes.c_int64), ("scale_bytes", ctypes.c_int64),
                ("aux_bytes", ctypes.c_int64), ("total_bytes", ctypes.c_int64), ("data", ctypes.c_void_p)]


_P = ctypes.c_void_p
_I = ctypes.c_int32
_L = ctypes.c_int64
_F = ctypes.c_float
_D = ctypes.POINTER(QTensorDesc)

# name -> argtypes (all functions return int status unless listed in _RESTYPES)
SIGNATURES = {
    "pmpd_version": [ctypes.POINTER(_I), ctypes.POINTER(_I)],
    "pmpd_last_error": [],
    "pmpd_qtensor_describe": [_I, _I, _I, _I, _I, _D],
    "pmpd_quantize": [_P, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P],
    "pmpd_planes_from_codes": [_P, _I, _I, _I, _P, _P],
    "pmpd_pack": [_D, _P, _P, _P, _P],
    "pmpd_unpack": [_D, _P, _P, _P, _P],
    "pmpd_prefix_codes": [_D, _I, _P, _P],
    "pmpd_dequant": [_D, _I, _P, _P],
    "pmpd_gather_rows": [_D, _P, _I, _P, _P, _P],
    "pmpd_gemv_workspace_bytes": [_D, _I, ctypes.POINTER(_L)],
    "pmpd_gemv": [_D, _P, _I, _I, _P, _P, _I, _I, _F, _I, _P, _L, _P],
    "pmpd_gemv_fused": [_D, _I, _P, _I, _I, _P, _F, _I, _P, _P, _I, _I, _F, _I, _P, _L, _P],
    "pmpd_gemm": [_D, _P, _I, _I, _P, _P, _I, _I, _F, _I, _P, _P],
    "pmpd_sched_step": [_P, _I, _P, _P, _I, _P],
    "pmpd_rmsnorm": [_P, _I, _P, _I, _I, _F, _P, _I, _P],
    "pmpd_rope_kv": [_P, _I, _I, _I, _I, _P, _P, _P, _I, _P, _P, _P, _P],
    "pmpd_attention": [_P, _I, _I, _I, _P, _P, _P, _I, _F, _P, _P],
    "pmpd_attention_rope": [_P, _I, _I, _P, _P, _P, _I, _F, _P, _P, _P, _P],
    "pmpd_attention_rope_batch": [_P, _I, _I, _I, _I, _P, _P, _P, _I, _F, _P, _P, _L, _P, _P],
    "pmpd_silu_mul": [_P, _I, _I, _I, _P, _I, _P],
    "pmpd_argmax": [_P, _I, _I, _I, _P, _P, _P],
    "pmpd_add_i32": [_P, _I, _P],
    "pmpd_push_token": [_P, _P, _P, _P, _I, _P],
    "pmpd_store_row": [_P, _P, _P, _I, _I, _P],
    "pmpd_engine_op_bytes": [],
    "pmpd_engine_grid": [],
    "pmpd_engine_max_slots": [_D],
    "pmpd_engine_nslots": [_D, _P],
    "pmpd_engine_make_op": [_D, _I, _I, _I, _I, _F, _P, _I, _P, _P],
    "pmpd_engine_run": [_P, _I, _P, _P, _P, _F, _P, _P, _P],
    "pmpd_engine_op_set_io": [_P, _I, _P, _P, _F, _I, _F],
    "pmpd_engine_make_attn_op": [_I, _I, _I, _P, _P, _P, _P, _P, _I, _F, _P, _P],
    "pmpd_engine_attn_records": [_I, _I],
    "pmpd_engine_partition": [_D, _P],
    "pmpd_engine_partition_g": [_D, _I, _P],
    "pmpd_engine_partition_w": [_D, _I, _P, _P],
    "pmpd_engine_run_ranks": [_P, _I, _I, _P, _P, _P, _I, _F, _P, _P, _P],
    "pmpd_engine_op_set_peers": [_P, _P, _I, _I],
    "pmpd_engine_op_set_bounds": [_P, _P],
    "pmpd_engine_op_set_counted": [_P, _P, _P, _I],
    "pmpd_engine_op_set_slice": [_P, _I, _I, _I, _I],
    "pmpd_engine_op_set_share": [_P, _I],
    "pmpd_engine_link": [_P, _I],
    "pmpd_engine_run_traced": [_P, _I, _P, _P, _P, _F, _P, _P, _P, _P],
    "pmpd_engine_run_decoder": [_P, _I, _P, _P, _P, _L, _I, _P, _F, _P, _P, _P, _P],
    "pmpd_engine_op_set_residual": [_P, _P, _I],
    "pmpd_learned_predict": [_P, _P, _I, _P, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _I, _I, _P, _P, _P],
}
_RESTYPES = {"pmpd_last_error": ctypes.c_char_p}

_lock = threading.Lock()
_lib = None


def lib():
    """Load the library once; raises ImportError (loudly) if it was not built."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise ImportError(f"PMPD CUDA library not built: {LIB_PATH} is missing "
                                      "(run __graft_entry__.build() or make -C paper_2410_13461_b200/csrc)")
                handle = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
                for name, args in SIGNATURES.items():
                    fn = getattr(handle, name)
                    fn.argtypes = args
                    fn.restype = _RESTYPES.get(name, ctypes.c_int)
                _lib = handle
    return _lib


def exported_symbols() -> list:
    return list(SIGNATURES)


def check(status: int, what: str = "") -> None:
    if status != OK:
        msg = lib().pmpd_last_error().decode("utf-8", "replace")
        raise _ERRORS.get(status, PmpdError)(f"{what}: {msg}" if what else msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)


def describe(rows: int, cols: int, group_size: int, p_max: int, layout: int) -> QTensorDesc:
    d = QTensorDesc()
    call("pmpd_qtensor_describe", rows, cols, group_size, p_max, layout, ctypes.byref(d))
    return d
