"""Loader of the in-tree sm_100a library (``libosmx_b200.so``) and its C-ABI.

The library is the product: there is no CPU fallback.  If the shared object
is missing or does not load, every entry point raises ``OsmxLibraryError``.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libosmx_b200.so"
# Diagnostic builds only (tools/c5_timeline.py sets it to build/tl/...)
if os.environ.get("OSMX_LIB_DIAG"):
    LIB_PATH = Path(os.environ["OSMX_LIB_DIAG"]).resolve()

# C-ABI status codes (include/osmx_b200.h)
(OK, ERR_EMPTY, ERR_NON_FINITE, ERR_INVALID_K, ERR_INVALID_CHUNK, ERR_INVALID_ARG, ERR_CUDA, ERR_UNSUPPORTED,
 ERR_NCCL) = range(9)

# Algorithm ids (include/osmx_b200.h, reference counting.hpp:17-24 order)
NAIVE_SOFTMAX = 0
SAFE_SOFTMAX = 1
ONLINE_SOFTMAX = 2
SAFE_SOFTMAX_UNFUSED_TOPK = 3
SAFE_SOFTMAX_FUSED_TOPK = 4
ONLINE_SOFTMAX_FUSED_TOPK = 5
ONLINE_SOFTMAX_UNFUSED_TOPK = 6

MAX_K = 32

# Every symbol include/osmx_b200.h declares: (name, restype, argtypes).
_vp, _sz, _i64, _i32, _int = C.c_void_p, C.c_size_t, C.c_int64, C.c_int32, C.c_int
_pi64 = C.POINTER(C.c_int64)
SIGNATURES = {
    "osmx_version": (_int, []),
    "osmx_status_string": (C.c_char_p, [_int]),
    "osmx_last_cuda_error": (C.c_char_p, []),
    "osmx_workspace_bytes": (_sz, [_int, _i64, _i64, _i32]),
    "osmx_workspace_init": (_int, [_vp, _sz, _vp]),
    "osmx_check_status": (_int, [_vp, _vp, _pi64]),
    "osmx_softmax": (_int, [_int, _vp, _i64, _vp, _i64, _i64, _i64, _vp, _sz, _vp]),
    "osmx_softmax_topk": (_int, [_int, _vp, _i64, _i64, _i64, _i32, _vp, _vp, _vp, _sz, _vp]),
    "osmx_topk": (_int, [_vp, _i64, _i64, _i64, _i32, _vp, _vp, _vp, _sz, _vp]),
    "osmx_normalizer": (_int, [_vp, _i64, _i64, _i64, _i64, _vp, _vp, _vp, _sz, _vp]),
    "osmx_normalizer_f64": (_int, [_vp, _i64, _i64, _i64, _i64, _vp, _vp, _vp, _sz, _vp]),
    "osmx_normalizer_workspace_bytes": (_sz, [_i64, _i64, _i64, _i32]),
    "osmx_normalizer_host": (_int, [_vp, _i64, _i64, _i64, _i32, _vp, _vp, _vp, _i32, _pi64]),
    "osmx_record_bytes": (_sz, [_i32]),
    "osmx_slice_record": (_int, [_vp, _i64, _i64, _i32, _vp, _vp, _sz, _vp]),
    "osmx_proj_softmax_topk": (_int, [_vp, _i64, _i64, _vp, _i64, _i32, _vp, _vp, _vp, _sz, _vp]),
    "osmx_records_combine": (_int, [_vp, _i32, _i32, _vp, _vp, _vp, _vp, _sz, _vp]),
    "osmx_scale_with_record": (_int, [_vp, _i64, _vp, _vp, _vp]),
    "osmx_softmax_host": (_int, [_int, _vp, _i64, _i64, _vp, _int, _pi64]),
    "osmx_softmax_topk_host": (_int, [_int, _vp, _i64, _i64, _i32, _vp, _vp, _int, _pi64]),
    "osmx_topk_host": (_int, [_vp, _i64, _i64, _i32, _vp, _vp, _int, _pi64]),
    "osmx_softmax_host_multi": (_int, [_int, _vp, _i64, _i64, _vp, _vp, _i32, _pi64]),
    "osmx_softmax_topk_host_multi": (_int, [_int, _vp, _i64, _i64, _i32, _vp, _vp, _vp, _i32, _pi64]),
    "osmx_topk_host_multi": (_int, [_vp, _i64, _i64, _i32, _vp, _vp, _vp, _i32, _pi64]),
    "osmx_host_release": (None, []),
    "osmx_launch_count": (C.c_uint64, []),
    "osmx_diag_read_probe": (_int, [_vp, _sz, _vp, _vp]),
    "osmx_config_set": (_int, [C.c_char_p, _i64]),
    "osmx_config_get": (_i64, [C.c_char_p]),
    "osmx_nccl_available": (_int, []),
    "osmx_last_nccl_error": (C.c_char_p, []),
    "osmx_nccl_get_unique_id": (_int, [_vp]),
    "osmx_nccl_comm_init": (_int, [C.POINTER(_vp), _i32, _vp, _i32]),
    "osmx_nccl_comm_destroy": (_int, [_vp]),
    "osmx_vsplit_workspace_bytes": (_sz, [_i64, _i32, _i32]),
    "osmx_vsplit_softmax_topk": (_int, [_vp, _i64, _i64, _i32, _vp, _vp, _vp, _vp, _sz, _vp]),
    "osmx_vsplit_softmax": (_int, [_vp, _i64, _i64, _vp, _vp, _vp, _sz, _vp]),
}


class OsmxLibraryError(RuntimeError):
    """The CUDA library is missing or failed to load (no fallback exists)."""


_lib = None


def load() -> C.CDLL:
    """Load ``libosmx_b200.so`` once; raise loudly if it is unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise OsmxLibraryError(
            f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
            "there is no CPU fallback")
    try:
        lib = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | getattr(os, "RTLD_GLOBAL", 0))
    except OSError as e:  # pragma: no cover - depends on the box
        raise OsmxLibraryError(f"cannot load {LIB_PATH}: {e}") from e
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def status_string(code: int) -> str:
    return load().osmx_status_string(code).decode()


def launch_count() -> int:
    return int(load().osmx_launch_count())


def config_set(key: str, value: int) -> None:
    st = load().osmx_config_set(key.encode(), int(value))
    if st != OK:
        raise ValueError(f"osmx_config_set({key!r}, {value}): {status_string(st)}")


def config_get(key: str) -> int:
    return int(load().osmx_config_get(key.encode()))
