"""ctypes binding of libhsv.so (the C ABI declared in include/hsv.h).

This is the only place Python touches native code.  There is no fallback:
if the library is missing or no sm_100 device is present, calls raise.
Status codes are mapped to the exception types the reference raises
(ValueError / RuntimeError / MemoryError) with the library's message.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "libhsv.so"

HSV_OK = 0
_ERRORS = {
    1: ValueError,    # HSV_ERR_INVALID
    2: ValueError,    # HSV_ERR_SECTOR
    3: ValueError,    # HSV_ERR_NONREAL
    4: ValueError,    # HSV_ERR_LEAK
    5: RuntimeError,  # HSV_ERR_NORM_DRIFT
    6: RuntimeError,  # HSV_ERR_CUDA
    7: MemoryError,   # HSV_ERR_OOM
    8: ValueError,    # HSV_ERR_UNSUPPORTED
}

i64, u64, dbl, vp = C.c_int64, C.c_uint64, C.c_double, C.c_void_p
P_i64, P_u64, P_dbl = C.POINTER(i64), C.POINTER(u64), C.POINTER(dbl)

# name: (restype, argtypes)
_SIGNATURES = {
    "hsv_abi_version": (C.c_int, []),
    "hsv_last_error": (C.c_int, [C.c_char_p, C.c_size_t]),
    "hsv_init": (C.c_int, [C.c_int]),
    "hsv_set_stream": (C.c_int, [vp]),
    "hsv_get_stream": (vp, []),
    "hsv_launch_count": (i64, [C.c_int]),
    "hsv_stats": (C.c_int, [P_i64, C.c_int]),
    "hsv_mem_trim": (C.c_int, []),
    "hsv_op_sell_info": (C.c_int, [vp, i64, i64, P_i64, P_i64]),
    "hsv_synchronize": (C.c_int, []),
    "hsv_sector_create": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(vp)]),
    "hsv_sector_destroy": (C.c_int, [vp]),
    "hsv_sector_dim": (i64, [vp]),
    "hsv_sector_shape": (C.c_int, [vp, P_i64, P_i64]),
    "hsv_sector_positions": (C.c_int, [vp, P_u64, i64, P_i64]),
    "hsv_sector_keys": (C.c_int, [vp, P_i64, i64, P_u64]),
    "hsv_op_create": (C.c_int, [vp, C.c_int, P_i64, P_i64, P_dbl, i64, C.POINTER(vp)]),
    "hsv_op_destroy": (C.c_int, [vp]),
    "hsv_op_info": (C.c_int, [vp, P_i64, P_i64, P_i64]),
    "hsv_op_count_nnz": (C.c_int, [vp, P_i64]),
    "hsv_op_to_csr": (C.c_int, [vp, P_i64, P_i64, P_dbl, i64]),
    "hsv_state_create": (C.c_int, [vp, C.POINTER(vp)]),
    "hsv_state_destroy": (C.c_int, [vp]),
    "hsv_state_copy": (C.c_int, [vp, vp]),
    "hsv_state_zero": (C.c_int, [vp]),
    "hsv_state_set_basis": (C.c_int, [vp, u64, dbl, dbl]),
    "hsv_state_set_sparse": (C.c_int, [vp, P_i64, P_dbl, P_dbl, i64]),
    "hsv_state_set_dense": (C.c_int, [vp, P_dbl, P_dbl]),
    "hsv_state_set_keys": (C.c_int, [vp, P_u64, P_dbl, P_dbl, i64]),
    "hsv_state_nnz": (C.c_int, [vp, P_i64]),
    "hsv_state_get_sparse": (C.c_int, [vp, dbl, P_i64, P_dbl, P_dbl, i64, P_i64]),
    "hsv_state_get_positions": (C.c_int, [vp, P_i64, i64, P_dbl, P_dbl]),
    "hsv_state_dot": (C.c_int, [vp, vp, P_dbl, P_dbl]),
    "hsv_state_norm": (C.c_int, [vp, P_dbl]),
    "hsv_state_axpy": (C.c_int, [dbl, dbl, vp, vp]),
    "hsv_state_scale": (C.c_int, [vp, dbl, dbl]),
    "hsv_apply_h": (C.c_int, [vp, vp, vp, dbl]),
    "hsv_expect_h": (C.c_int, [vp, vp, P_dbl, P_dbl]),
    "hsv_apply_qeb": (C.c_int, [vp, vp, u64, u64, dbl, dbl]),
    "hsv_ansatz_state": (C.c_int, [vp, u64, P_u64, P_u64, P_dbl, P_dbl, i64, vp]),
    "hsv_apply_generator": (C.c_int, [vp, vp, u64, u64]),
    "hsv_energy_screen": (C.c_int, [vp, vp, P_u64, P_u64, i64, P_dbl, P_dbl]),
    "hsv_energy_gradient": (C.c_int, [vp, u64, P_u64, P_u64, P_dbl, P_dbl, i64, P_dbl, P_dbl]),
    "hsv_eg_forward_async": (C.c_int, [vp, u64, P_u64, P_u64, P_dbl, P_dbl, i64, i64, i64, vp,
                                       vp]),
    "hsv_eg_backward": (C.c_int, [vp, vp, vp, P_u64, P_u64, P_dbl, P_dbl, i64, P_dbl, P_dbl]),
    "hsv_energy_screen_partial_async": (C.c_int, [vp, vp, P_u64, P_u64, i64, i64, i64, vp]),
    "hsv_state_device_ptr": (C.c_int, [vp, C.POINTER(vp), P_i64]),
    "hsv_apply_h_rows_async": (C.c_int, [vp, vp, vp, i64, i64, dbl]),
    "hsv_csr_spmspv": (C.c_int, [i64, i64, P_i64, P_i64, P_dbl, i64, P_i64, P_dbl, i64, dbl,
                                 P_i64, P_dbl, P_i64]),
    "hsv_vec_dot": (C.c_int, [P_i64, P_dbl, i64, P_i64, P_dbl, i64, P_dbl]),
    "hsv_vec_axpy": (C.c_int, [i64, dbl, P_i64, P_dbl, i64, P_i64, P_dbl, i64, dbl, P_i64,
                               P_dbl, P_i64]),
    "hsv_vec_scale": (C.c_int, [P_dbl, i64, dbl, C.c_int, P_dbl]),
    "hsv_pool_create": (C.c_int, [vp, P_u64, P_u64, i64, C.POINTER(vp)]),
    "hsv_pool_destroy": (C.c_int, [vp]),
    "hsv_energy_screen_pool_async": (C.c_int, [vp, vp, vp, i64, i64, vp]),
    "hsv_energy_screen_pool": (C.c_int, [vp, vp, vp, P_dbl, P_dbl]),
    "hsv_sum_rows_async": (C.c_int, [vp, i64, i64, vp]),
    "hsv_peer_create": (C.c_int, [C.c_int, C.c_int, i64, C.POINTER(vp), vp]),
    "hsv_peer_open": (C.c_int, [vp, vp]),
    "hsv_peer_destroy": (C.c_int, [vp]),
    "hsv_peer_check": (C.c_int, [vp]),
    "hsv_peer_data": (C.c_int, [vp, C.POINTER(vp), C.POINTER(i64)]),
    "hsv_peer_allgather_async": (C.c_int, [vp, vp, i64]),
    "hsv_peer_allreduce_async": (C.c_int, [vp, vp, i64, vp]),
    "hsv_eg_forward_peer_async": (C.c_int, [vp, C.c_uint64, P_u64, P_u64, P_dbl, P_dbl, i64,
                                            i64, i64, vp, vp, vp]),
    "hsv_set_tuning": (C.c_int, [C.c_char_p, i64]),
    "hsv_jordan_wigner": (C.c_int, [C.c_int, P_dbl, P_dbl, dbl, dbl, P_i64, P_i64, P_dbl, i64,
                                    P_i64]),
    "hsv_krylov_project": (C.c_int, [C.POINTER(vp), i64, vp, C.c_int, P_dbl]),
    "hsv_krylov_combine": (C.c_int, [C.POINTER(vp), i64, P_dbl, vp]),
    "hsv_prof_enable": (C.c_int, [C.c_int]),
    "hsv_prof_collect": (C.c_int, []),
    "hsv_prof_get": (C.c_int, [C.c_char_p, P_dbl, P_i64]),
    "hsv_prof_reset": (C.c_int, []),
}

_lib = None
_lock = threading.Lock()


def load(path: str | os.PathLike | None = None) -> C.CDLL:
    """Load libhsv.so (raises OSError when it has not been built)."""
    global _lib
    with _lock:
        if _lib is None:
            p = Path(path) if path else LIB_PATH
            if not p.exists():
                raise OSError(f"libhsv.so not found at {p}; run __graft_entry__.build() "
                              "(the CUDA path has no CPU fallback)")
            lib = C.CDLL(str(p))
            for name, (res, args) in _SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
        return _lib


def exported_symbols() -> list[str]:
    return list(_SIGNATURES)


def lib() -> C.CDLL:
    return _lib if _lib is not None else load()


def check(rc: int):
    if rc != HSV_OK:
        buf = C.create_string_buffer(2048)
        lib().hsv_last_error(buf, len(buf))
        raise _ERRORS.get(rc, RuntimeError)(buf.value.decode(errors="replace"))


def call(name: str, *args):
    check(getattr(lib(), name)(*args))


_device = None


def init(device: int | None = None):
    """Bind the library to a CUDA device (default: current torch device or 0)."""
    global _device
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", "0")) if _device is None else _device
    if _device != device:
        call("hsv_init", int(device))
        _device = device
    return _device


# ----------------------------------------------------------- array helpers
def ptr_i64(a: np.ndarray):
    return a.ctypes.data_as(P_i64)


def ptr_u64(a: np.ndarray):
    return a.ctypes.data_as(P_u64)


def ptr_f64(a: np.ndarray):
    return a.ctypes.data_as(P_dbl)


def as_i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def as_u64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a).astype(np.uint64, copy=False))


def as_f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)
