"""ctypes binding of libspf.so (include/spf.h).

The library is built in-tree by ``paper_2407_02490_b200.build`` (or
``__graft_entry__.build()``).  There is deliberately no fallback: if the
library is missing or cannot be loaded, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libspf.so")

SPF_DTYPE_BF16 = 0
SPF_DTYPE_F32 = 1
SPF_VS_EXACT = 0
SPF_VS_FAST = 1
SPF_VS_FAST_UNCERTIFIED = 2  # test hook: tensor-core path without re-estimation (not exact)

_c_int = ctypes.c_int
_c_float = ctypes.c_float
_c_size = ctypes.c_size_t
_vp = ctypes.c_void_p
_i64 = ctypes.c_int64

# name -> (restype, argtypes); mirrors include/spf.h one-to-one.
SIGNATURES = {
    "spf_version": (_c_int, []),
    "spf_last_error": (ctypes.c_char_p, []),
    "spf_kernel_launches": (ctypes.c_ulonglong, []),
    "spf_sparse_flash_workspace_size": (_c_size, [_c_int, _c_int, _c_int, _c_int, _c_int]),
    "spf_sparse_flash_rows": (_c_int, [_c_int, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_float, _c_int,
                                       _vp, _vp, _vp, _vp, _vp, _vp, _c_size, _vp]),
    "spf_sparse_flash_rows_lse": (_c_int, [_c_int, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_float, _c_int,
                                           _vp, _vp, _vp, _vp, _vp, _vp, _vp, _c_size, _vp]),
    "spf_sparse_flash_rows_ex": (_c_int, [_c_int, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_float, _c_int,
                                          _vp, _vp, _vp, _vp, _vp, _c_int, _vp, _vp, _vp, _c_size, _vp]),
    "spf_argtopk_workspace_size": (_c_size, [_i64]),
    "spf_argtopk": (_c_int, [_vp, _i64, _c_int, _vp, _vp, _c_size, _vp]),
    "spf_vs_estimate_workspace_size": (_c_size, [_c_int] * 8),
    "spf_vs_estimate": (_c_int, [_c_int, _c_int, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _vp, _c_int, _c_int, _c_int,
                                 _c_int, _vp, _vp, _vp, _vp, _vp, _vp, _c_size, _vp]),
    "spf_bs_estimate_workspace_size": (_c_size, [_c_int, _c_int, _c_int, _c_int, _c_int]),
    "spf_bs_estimate": (_c_int, [_c_int, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _vp, _c_int, _c_int, _c_int,
                                 _vp, _vp, _vp, _c_size, _vp]),
    "spf_scan_workspace_size": (_c_size, [_i64]),
    "spf_csr_offsets": (_c_int, [_vp, _i64, _vp, _vp, _vp, _c_size, _vp]),
    "spf_csr_guard": (_c_int, [_vp, _vp, _i64, _i64, _i64, _vp, _vp, _vp]),
    "spf_vs_layout_count": (_c_int, [_vp, _c_int, _vp, _c_int, _vp, _c_int, _c_int, _c_int, _vp, _vp, _vp]),
    "spf_vs_layout_fill": (_c_int, [_vp, _c_int, _vp, _c_int, _vp, _c_int, _c_int, _c_int, _vp, _vp, _vp, _vp,
                                    _vp]),
    "spf_ashape_layout_count": (_c_int, [_vp, _c_int, _c_int, _c_int, _c_int, _c_int, _vp, _vp]),
    "spf_ashape_layout_fill": (_c_int, [_vp, _c_int, _c_int, _c_int, _c_int, _c_int, _vp, _vp, _vp]),
    "spf_bs_layout_count": (_c_int, [_vp, _c_int, _c_int, _c_int, _c_int, _vp, _vp]),
    "spf_layout_area": (_c_int, [_c_int, _c_int, _c_int, _vp, _vp, _vp, _vp, _vp]),
    "spf_f32_to_bf16": (_c_int, [_vp, _vp, _i64, _vp]),
}


class SpfError(RuntimeError):
    """A libspf call returned a non-zero status."""


_lib = None


def load():
    """Load (once) and return the configured ctypes library handle."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} not found: build it with `python -m paper_2407_02490_b200.build` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    missing = []
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name, None)
        if fn is None:
            missing.append(name)
            continue
        fn.restype = res
        fn.argtypes = args
    lib.spf_missing_symbols = missing
    _lib = lib
    return lib


def missing_symbols() -> list:
    """Entry points declared in include/spf.h but absent from the library."""
    return list(load().spf_missing_symbols)


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = load().spf_last_error().decode(errors="replace")
        if rc == 2:
            raise ValueError(f"{what}: {msg}")
        raise SpfError(f"{what} failed (code {rc}): {msg}")


def call(name: str, *args):
    lib = load()
    rc = getattr(lib, name)(*args)
    check(rc, name)
    return rc
