"""ctypes loader for libhaarshift.so (the C ABI declared in include/haarshift.h).

The product path has exactly one implementation: the CUDA kernels behind this library.  If the
library is missing or cannot be loaded, every call raises -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libhaarshift.so")

# name -> (restype, argtypes); mirrors include/haarshift.h
_c = ctypes
SIGNATURES = {
    "haar_shift_coeffs": (_c.c_int, [_c.c_void_p, _c.c_void_p, _c.c_int, _c.c_int, _c.c_int, _c.c_int,
                                     _c.c_void_p, _c.c_int, _c.c_void_p, _c.c_size_t, _c.c_void_p]),
    "haar_shift_workspace_bytes": (_c.c_size_t, [_c.c_int, _c.c_int, _c.c_int, _c.c_int]),
    "haar_shift_coeffs_coarse": (_c.c_int, [_c.c_void_p, _c.c_void_p, _c.c_int, _c.c_int, _c.c_int, _c.c_int,
                                            _c.c_void_p, _c.c_int, _c.c_void_p, _c.c_size_t, _c.c_void_p]),
    "haar_shift_coarse_workspace_bytes": (_c.c_size_t, [_c.c_int, _c.c_int, _c.c_int, _c.c_int]),
    "relight_vertices": (_c.c_int, [_c.c_void_p, _c.c_int64, _c.c_int, _c.c_int, _c.c_void_p, _c.c_int64,
                                    _c.c_int, _c.c_void_p, _c.c_void_p, _c.c_size_t, _c.c_void_p]),
    "relight_workspace_bytes": (_c.c_size_t, [_c.c_int, _c.c_int, _c.c_int]),
    "relight_vertices_shifted": (_c.c_int, [_c.c_void_p, _c.c_int64, _c.c_int, _c.c_void_p, _c.c_int,
                                            _c.c_void_p, _c.c_void_p, _c.c_void_p, _c.c_size_t, _c.c_void_p]),
    "relight_shifted_workspace_bytes": (_c.c_size_t, [_c.c_int64, _c.c_int, _c.c_int]),
    "hs_fill_transfer": (_c.c_int, [_c.c_void_p, _c.c_int64, _c.c_int64, _c.c_int, _c.c_int, _c.c_uint64,
                                    _c.c_uint64, _c.c_void_p]),
    "relight_vertices_sparse": (_c.c_int, [_c.c_void_p, _c.c_void_p, _c.c_int64, _c.c_int, _c.c_void_p, _c.c_int64,
                                           _c.c_int, _c.c_void_p, _c.c_void_p, _c.c_size_t, _c.c_void_p]),
    "relight_sparse_workspace_bytes": (_c.c_size_t, [_c.c_int64, _c.c_int]),
    "hs_fill_sparse_transfer": (_c.c_int, [_c.c_void_p, _c.c_void_p, _c.c_int64, _c.c_int64, _c.c_int, _c.c_int,
                                           _c.c_int, _c.c_int, _c.c_uint64, _c.c_void_p]),
    "relight_vertices_triple": (_c.c_int, [_c.c_void_p, _c.c_void_p, _c.c_int64, _c.c_int, _c.c_int, _c.c_void_p,
                                           _c.c_int64, _c.c_int, _c.c_void_p, _c.c_void_p, _c.c_size_t, _c.c_void_p]),
    "relight_triple_workspace_bytes": (_c.c_size_t, [_c.c_int64, _c.c_int, _c.c_int, _c.c_int]),
    "haar_pack_qtree": (_c.c_int, [_c.c_void_p, _c.c_int64, _c.c_int, _c.c_int64, _c.c_int, _c.c_void_p,
                                   _c.c_void_p]),
    "relight_vertices_brdf_rotated": (_c.c_int, [_c.c_void_p, _c.c_int, _c.c_void_p, _c.c_int64, _c.c_void_p, _c.c_int,
                                                 _c.c_void_p, _c.c_int64, _c.c_int, _c.c_void_p, _c.c_void_p,
                                                 _c.c_size_t, _c.c_void_p]),
    "relight_brdf_rotated_workspace_bytes": (_c.c_size_t, [_c.c_int, _c.c_int, _c.c_int]),
    "haar_rotate_coeffs": (_c.c_int, [_c.c_void_p, _c.c_void_p, _c.c_int, _c.c_int, _c.c_void_p, _c.c_void_p,
                                      _c.c_size_t, _c.c_void_p]),
    "haar_rotate_workspace_bytes": (_c.c_size_t, [_c.c_int, _c.c_int]),
    "hs_enable_peer_access": (_c.c_int, [_c.c_int]),
    "hs_last_launch_count": (_c.c_int, []),
    "hs_status_string": (_c.c_char_p, [_c.c_int]),
    "hs_last_cuda_error": (_c.c_char_p, []),
    "hs_abi_version": (_c.c_int, []),
}

STATUS = {0: "HS_OK", 1: "HS_ERR_INVALID_ARG", 2: "HS_ERR_ALIGNMENT", 3: "HS_ERR_UNSUPPORTED", 4: "HS_ERR_CUDA"}


class HaarShiftError(RuntimeError):
    def __init__(self, fn: str, status: int, detail: str = ""):
        self.status = status
        msg = f"{fn} failed: {STATUS.get(status, status)}"
        if detail:
            msg += f" ({detail})"
        super().__init__(msg)


_LIB = None


def load() -> ctypes.CDLL:
    """Load libhaarshift.so once; raise loudly if it is missing (build with __graft_entry__.build())."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libhaarshift.so not built at {LIB_PATH}; run python -c 'import __graft_entry__ as g; "
                          "g.build()' (there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def check(fn: str, status: int) -> None:
    if status != 0:
        detail = ""
        if status == 4 or status == 3:
            detail = (load().hs_last_cuda_error() or b"").decode(errors="replace")
        raise HaarShiftError(fn, status, detail)
