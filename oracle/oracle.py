"""ctypes face of the CPU checkers.  TEST INFRASTRUCTURE ONLY.

Two libraries, both built by ``oracle/Makefile``:

* ``port`` -- ``_build/libosmx_oracle.so``: our plain-C restatement of the
  reference algorithms (``osmx_oracle.c``; every function cites the
  reference file:line it follows).
* ``ref``  -- ``_ref/libosmx_ref.so``: the unmodified reference library
  (``/root/reference/proj/src``) compiled with ``-Dosmx=osmx_ref`` behind an
  ``extern "C"`` shim (``ref_shim.cpp``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module.  The
product path (``paper_1805_02867_b200``) never does.

Parity of the port is pinned by ``tests/test_oracle.py`` (bit-exact against
``ref`` and against the frozen constants of
``/root/reference/proj/tests/test_support.hpp:47-56``).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_SO = HERE / "_build" / "libosmx_oracle.so"
REF_SO = HERE / "_ref" / "libosmx_ref.so"

# Status codes shared by both libraries (reference error.hpp:8-25).
OK, EMPTY, NON_FINITE, INVALID_K, INVALID_CHUNK = 0, 1, 2, 3, 4

# Batched op codes (ref_shim.cpp / osmx_oracle.c oracle_batch).
OPS = {
    "naive_softmax": 0,
    "safe_softmax": 1,
    "online_softmax": 2,
    "safe_softmax_then_topk": 3,
    "safe_softmax_fused_topk": 4,
    "online_softmax_topk": 5,
    "topk_of": 6,
    "oracle_topk": 7,
}
TOPK_OPS = {"safe_softmax_then_topk", "safe_softmax_fused_topk", "online_softmax_topk", "topk_of", "oracle_topk"}

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")

_port = None
_ref = None


def build() -> None:
    """Compile the checkers (the port always; the reference when its sources exist)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def port():
    global _port
    if _port is None:
        if not PORT_SO.exists():
            build()
        lib = C.CDLL(str(PORT_SO))
        for name in ("oracle_naive_softmax", "oracle_safe_softmax", "oracle_online_softmax"):
            f = getattr(lib, name)
            f.argtypes = [_f32p, C.c_size_t, _f32p]
            f.restype = C.c_int
        for name in ("oracle_topk_of", "oracle_safe_softmax_then_topk", "oracle_safe_softmax_fused_topk",
                     "oracle_online_softmax_topk", "oracle_topk_sort"):
            f = getattr(lib, name)
            f.argtypes = [_f32p, C.c_size_t, C.c_size_t, _f32p, _i64p]
            f.restype = C.c_int
        lib.oracle_softmax_double.argtypes = [_f32p, C.c_size_t, _f64p]
        lib.oracle_softmax_double.restype = C.c_int
        lib.oracle_normalizer_double.argtypes = [_f32p, C.c_size_t, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        lib.oracle_normalizer_double.restype = C.c_int
        lib.oracle_run_normalizer.argtypes = [_f32p, C.c_size_t, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        lib.oracle_run_normalizer.restype = C.c_int
        lib.oracle_run_normalizer_chunked.argtypes = [_f32p, C.c_size_t, C.c_size_t, C.c_int,
                                                      C.POINTER(C.c_double), C.POINTER(C.c_double)]
        lib.oracle_run_normalizer_chunked.restype = C.c_int
        lib.oracle_merge_d.argtypes = [C.c_double] * 4 + [C.POINTER(C.c_double)] * 2
        lib.oracle_merge_d.restype = None
        lib.oracle_merge_f.argtypes = [C.c_float] * 4 + [C.POINTER(C.c_float)] * 2
        lib.oracle_merge_f.restype = None
        lib.oracle_count_accesses.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64),
                                              C.POINTER(C.c_uint64)]
        lib.oracle_count_accesses.restype = C.c_int
        lib.oracle_batch.argtypes = [C.c_int, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                     C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
        lib.oracle_batch.restype = C.c_int
        _port = lib
    return _port


def ref_available() -> bool:
    return REF_SO.exists()


def ref():
    global _ref
    if _ref is None:
        if not REF_SO.exists():
            raise RuntimeError(f"reference library not built: {REF_SO} (run make -C oracle)")
        lib = C.CDLL(str(REF_SO))
        lib.osmx_ref_row.argtypes = [C.c_int, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
        lib.osmx_ref_row.restype = C.c_int
        lib.osmx_ref_batch.argtypes = [C.c_int, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                       C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
        lib.osmx_ref_batch.restype = C.c_int
        lib.osmx_ref_oracle_softmax.argtypes = [_f32p, C.c_int64, _f64p]
        lib.osmx_ref_oracle_softmax.restype = C.c_int
        lib.osmx_ref_oracle_normalizer.argtypes = [_f32p, C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        lib.osmx_ref_oracle_normalizer.restype = C.c_int
        lib.osmx_ref_normalizer.argtypes = [_f32p, C.c_int64, C.c_int, C.c_int, C.c_int64,
                                            C.POINTER(C.c_double), C.POINTER(C.c_double)]
        lib.osmx_ref_normalizer.restype = C.c_int
        lib.osmx_ref_merge.argtypes = [C.c_int] + [C.c_double] * 4 + [C.POINTER(C.c_double)] * 2
        lib.osmx_ref_merge.restype = None
        lib.osmx_ref_generate_inputs.argtypes = [C.c_uint64, C.c_int64, C.c_int64, _f32p]
        lib.osmx_ref_generate_inputs.restype = C.c_int
        lib.osmx_ref_count_accesses.argtypes = [C.c_int, C.c_int64, C.c_int64, C.POINTER(C.c_uint64),
                                                C.POINTER(C.c_uint64)]
        lib.osmx_ref_count_accesses.restype = C.c_int
        lib.osmx_ref_log_spaced_sizes.argtypes = [C.c_int64, C.c_int64, C.c_int64, _i64p, C.c_int64]
        lib.osmx_ref_log_spaced_sizes.restype = C.c_int64
        lib.osmx_ref_sweep_cell.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                            C.c_uint64, C.c_int64]
        lib.osmx_ref_sweep_cell.restype = C.c_double
        _ref = lib
    return _ref


# ----------------------------------------------------------------- helpers --

def _rows(x) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    return x.reshape(1, -1) if x.ndim == 1 else x


def batch(op: str, x, k: int = 0, threads: int = 1, impl: str = "port"):
    """Run one entry point over every row of ``x`` (2-D, row-major).

    Returns (y, status) for softmax ops and (values, indices, status) for the
    top-K ops; status[r] is the per-row status code.
    """
    x = _rows(x)
    rows, n = x.shape
    st = np.zeros(rows, np.int32)
    code = OPS[op]
    if op in TOPK_OPS:
        v = np.zeros((rows, max(k, 1)), np.float32)
        z = np.zeros((rows, max(k, 1)), np.int64)
        y_ptr, ldy = None, 0
        v_ptr, z_ptr = v.ctypes.data, z.ctypes.data
    else:
        y = np.zeros((rows, n), np.float32)
        y_ptr, ldy = y.ctypes.data, n
        v_ptr = z_ptr = None
    if impl == "ref":
        ref().osmx_ref_batch(code, x.ctypes.data, n, rows, n, k, y_ptr, ldy, v_ptr, z_ptr, st.ctypes.data, threads)
    else:
        if code == 7:
            raise ValueError("oracle_topk is only exposed by the port via topk_sort()")
        port().oracle_batch(code, x.ctypes.data, n, rows, n, k, y_ptr, ldy, v_ptr, z_ptr, st.ctypes.data, threads)
    if op in TOPK_OPS:
        return v, z, st
    return y, st


def softmax(op: str, x, impl: str = "port"):
    """Single-row softmax; returns (y, status)."""
    y, st = batch(op, np.asarray(x, np.float32).reshape(1, -1), impl=impl)
    return y[0], int(st[0])


def topk(op: str, x, k: int, impl: str = "port"):
    """Single-row top-K; returns (values, indices, status)."""
    v, z, st = batch(op, np.asarray(x, np.float32).reshape(1, -1), k=k, impl=impl)
    return v[0], z[0], int(st[0])


def topk_sort(x, k: int):
    x = np.ascontiguousarray(x, np.float32).ravel()
    v = np.zeros(max(k, 1), np.float32)
    z = np.zeros(max(k, 1), np.int64)
    st = port().oracle_topk_sort(x, x.size, k, v, z)
    return v[:k], z[:k], st


def softmax_double(x, impl: str = "port"):
    x = np.ascontiguousarray(x, np.float32).ravel()
    y = np.zeros(max(x.size, 1), np.float64)
    if impl == "ref":
        st = ref().osmx_ref_oracle_softmax(x, x.size, y)
    else:
        st = port().oracle_softmax_double(x, x.size, y)
    return y[: x.size], st


def normalizer(x, dbl: bool = True, chunk: int | None = None, impl: str = "port"):
    """(m, d, status): run_normalizer / run_normalizer_chunked (normalizer.hpp:61-85)."""
    x = np.ascontiguousarray(x, np.float32).ravel()
    m, d = C.c_double(0), C.c_double(0)
    if impl == "ref":
        st = ref().osmx_ref_normalizer(x, x.size, int(dbl), int(chunk is not None), chunk or 0, C.byref(m), C.byref(d))
    elif chunk is None:
        st = port().oracle_run_normalizer(x, x.size, int(dbl), C.byref(m), C.byref(d))
    else:
        st = port().oracle_run_normalizer_chunked(x, x.size, chunk, int(dbl), C.byref(m), C.byref(d))
    return m.value, d.value, st


def merge(a, b, dbl: bool = True, impl: str = "port"):
    if impl == "ref":
        m, d = C.c_double(0), C.c_double(0)
        ref().osmx_ref_merge(int(dbl), a[0], a[1], b[0], b[1], C.byref(m), C.byref(d))
        return m.value, d.value
    if dbl:
        m, d = C.c_double(0), C.c_double(0)
        port().oracle_merge_d(a[0], a[1], b[0], b[1], C.byref(m), C.byref(d))
    else:
        m, d = C.c_float(0), C.c_float(0)
        port().oracle_merge_f(a[0], a[1], b[0], b[1], C.byref(m), C.byref(d))
    return m.value, d.value


def count_accesses(alg: int, v: int, k: int = 0, impl: str = "port"):
    lo, st_ = C.c_uint64(0), C.c_uint64(0)
    if impl == "ref":
        s = ref().osmx_ref_count_accesses(alg, v, k, C.byref(lo), C.byref(st_))
    else:
        s = port().oracle_count_accesses(alg, v, k, C.byref(lo), C.byref(st_))
    return lo.value, st_.value, s


def generate_inputs(seed: int, batch_: int, v: int) -> np.ndarray:
    """The reference's own generator (bench.cpp:162-172: mt19937_64 + normal_distribution<float>)."""
    out = np.zeros(batch_ * v, np.float32)
    st = ref().osmx_ref_generate_inputs(seed, batch_, v, out)
    if st:
        raise ValueError(f"generate_inputs status {st}")
    return out.reshape(batch_, v)


def log_spaced_sizes(vmin: int, vmax: int, points: int) -> list[int]:
    out = np.zeros(max(points, 1) + 4, np.int64)
    n = ref().osmx_ref_log_spaced_sizes(vmin, vmax, points, out, out.size)
    if n < 0:
        raise ValueError("log_spaced_sizes: invalid arguments")
    return [int(v) for v in out[:n]]


def host_threads() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
