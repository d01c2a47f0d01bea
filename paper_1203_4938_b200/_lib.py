"""ctypes binding of libdpp_b200.so (the C ABI in include/dpp_b200.h).

Loading is strict: if the library is missing or was built for another ABI
version the import of any node raises :class:`NativeLibraryError`.  There is
no CPU fallback anywhere in the product path.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from .errors import DeviceError, NativeLibraryError, PlanError

LIB_PATH = Path(os.environ.get("DPP_LIB_PATH") or Path(__file__).resolve().parent / "libdpp_b200.so")
ABI_VERSION = 1

DPP_OK, DPP_EINVAL, DPP_ECUDA, DPP_ENCCL, DPP_ENOTSUP = 0, 1, 2, 3, 4

_vp, _i64, _int, _sz = C.c_void_p, C.c_int64, C.c_int, C.c_size_t

# name -> (restype, argtypes); mirrors include/dpp_b200.h one to one
SIGNATURES = {
    "dpp_abi_version": (_int, []),
    "dpp_last_error": (C.c_char_p, []),
    "dpp_fft_plan_create": (_int, [C.POINTER(_vp), _int, _i64, _i64, _i64, C.POINTER(_sz)]),
    "dpp_fft_plan_describe": (_int, [_vp, C.c_char_p, _sz]),
    "dpp_fft_plan_supported": (_int, [_int, _i64, _i64]),
    "dpp_fft_c2c_forward": (_int, [_vp, _vp, _vp, _vp, _vp]),
    "dpp_fft_c2c_forward_batch": (_int, [_vp, _vp, _vp, _i64, _vp, _vp]),
    "dpp_fft_plan_destroy": (None, [_vp]),
    "dpp_fft_c2c_columns": (_int, [_vp, _vp, _i64, _vp]),
    "dpp_fft_twiddle": (_int, [_vp, _i64, _i64, _i64, _i64, _vp]),
    "dpp_fft_leaf": (_int, [_int, _vp, _vp, _i64, _vp]),
    "dpp_naive_dft": (_int, [_vp, _vp, _i64, _i64, _vp]),
    "dpp_imgc_ycbcr": (_int, [_vp, _vp, _vp, _vp, _i64, _vp]),
    "dpp_imgc_boxdown": (_int, [_vp, _vp, _i64, _vp]),
    "dpp_imgc_gradient": (_int, [_vp, _vp, _vp, _i64, _i64, _i64, C.POINTER(_i64), _vp]),
    "dpp_imgc_vqnearest": (_int, [_vp, _vp, _vp, _i64, _i64, _int, _vp]),
    "dpp_imgc_encode": (_int, [_vp, _int, _i64, _i64, _i64, _i64, _i64, _vp, _int, _i64,
                               C.c_double, _vp, _vp, _vp, _vp, _vp, _vp]),
    "dpp_imgc_encode_planar": (_int, [_vp, _int, _i64, _i64, _i64, _i64, _i64, _vp, _int, _i64,
                                      C.c_double, _vp, _vp, _vp, _vp, _vp, _vp]),
    "dpp_imgc_decode": (_int, [_vp, _vp, _vp, _vp, _int, _i64, _i64, _vp, _vp]),
    "dpp_imgc_encode_tc_debug": (_int, [_vp, _int, _i64, _i64, _vp, _int, _vp, _vp, _vp, C.c_float, _vp, _vp]),
    "dpp_u8_to_complex": (_int, [_vp, _vp, _i64, _vp]),
    "dpp_spectrum_u8": (_int, [_vp, _vp, _i64, C.c_float, _vp]),
    "dpp_imgc_block_stats": (_int, [_vp, _int, _i64, _i64, _i64, _i64, _i64, C.c_double, _vp, _vp, _vp]),
    "dpp_imgc_rounding_ties": (_int, [_vp, _int, _i64, _i64, _i64, _i64, _i64, _vp, _vp]),
    "dpp_kmeans": (_int, [_vp, _i64, _int, _i64, C.POINTER(C.c_double), _int, _vp,
                          C.POINTER(C.c_double), C.POINTER(_int), _vp]),
    "dpp_fft2d_u8_spectrum": (_int, [_vp, _vp, _vp, C.c_float, _vp, _i64, _vp]),
    "dpp_jit_compile": (_int, [C.c_char_p, C.c_char_p, C.POINTER(_vp), C.c_char_p, _sz]),
    "dpp_jit_launch": (_int, [_vp, C.POINTER(C.c_uint64), _int, _i64, _vp]),
    "dpp_jit_destroy": (None, [_vp]),
    "dpp_fft2d_columns_sharded": (_int, [_vp, C.POINTER(_vp), C.POINTER(_vp), _int, _int, _int, _i64, _vp]),
    "dpp_ipc_get_handle": (_int, [_vp, _vp, C.POINTER(C.c_uint64)]),
    "dpp_ipc_open": (_int, [_vp, C.POINTER(_vp)]),
    "dpp_ipc_close": (_int, [_vp]),
    "dpp_kmeans_shard_create": (_int, [C.POINTER(_vp), _vp, _i64, _int, _vp]),
    "dpp_kmeans_shard_seed": (_int, [_vp, _vp, _int, C.POINTER(C.c_double)]),
    "dpp_kmeans_shard_pick": (_int, [_vp, C.c_double, _i64, _vp, C.POINTER(_i64)]),
    "dpp_kmeans_shard_assign": (_int, [_vp, _vp, _vp]),
    "dpp_kmeans_shard_far": (_int, [_vp, _vp, _i64, _vp]),
    "dpp_kmeans_shard_set_assign": (_int, [_vp, _i64, _int]),
    "dpp_kmeans_shard_destroy": (None, [_vp]),
    "dpp_peer_group_create": (_int, [C.POINTER(_vp), _int, _int, C.POINTER(_vp), C.POINTER(_vp), C.c_double]),
    "dpp_peer_group_destroy": (None, [_vp]),
    "dpp_fft2d_c2c_fwd_sharded": (_int, [_vp, _vp, _vp, _vp, _int, _i64, _vp]),
    "dpp_peer_barrier": (_int, [C.POINTER(_vp), _int, _int, _int, C.c_double, _vp]),
}

_lock = threading.Lock()
_lib: C.CDLL | None = None


def load() -> C.CDLL:
    """Load (once) and type the library; raise NativeLibraryError if unusable."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise NativeLibraryError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                " (there is no CPU fallback)")
        try:
            lib = C.CDLL(str(LIB_PATH))
        except OSError as exc:
            raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.dpp_abi_version() != ABI_VERSION:
            raise NativeLibraryError(
                f"ABI version {lib.dpp_abi_version()} != expected {ABI_VERSION}; rebuild the library")
        _lib = lib
    return _lib


def last_error() -> str:
    return (load().dpp_last_error() or b"").decode("utf-8", "replace")


def check(rc: int, what: str = "") -> None:
    """Map a C-ABI return code onto the reference's exception classes."""
    if rc == DPP_OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if rc in (DPP_EINVAL, DPP_ENOTSUP):
        raise PlanError(msg)
    raise DeviceError(msg)


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None for None)."""
    return None if t is None else t.data_ptr()
