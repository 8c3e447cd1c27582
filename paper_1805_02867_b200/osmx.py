"""Python host API mirroring the reference ``osmx`` library, backed by the
sm_100a kernels through the C-ABI (include/osmx_b200.h).

Two layers:

* **Reference-shaped functions** (same names, argument meaning and error
  behaviour as ``proj/include/osmx/{softmax,topk,normalizer}.hpp``): a 1-D
  float vector in, a fresh result out.  They run the batched host-buffer
  entry points (``osmx_*_host``) -- copy in, kernel, copy out -- and accept a
  2-D array as a batch of rows.

    naive_softmax(x)             softmax.hpp:17   (Alg. 1)
    safe_softmax(x)              softmax.hpp:22   (Alg. 2)
    online_softmax(x)            softmax.hpp:28   (Alg. 3)
    topk_of(values, k)           topk.hpp:54
    safe_softmax_then_topk(x, k) topk.hpp:58
    safe_softmax_fused_topk(x,k) topk.hpp:63
    online_softmax_topk(x, k)    topk.hpp:68      (Alg. 4)
    run_normalizer(x)            normalizer.hpp:61-67
    run_normalizer_chunked(x,c)  normalizer.hpp:73-85

  Errors are the reference's exception types (error.hpp:8-25), all
  subclasses of ValueError as the reference's derive from
  std::invalid_argument.

* **Batched device functions** on torch CUDA tensors (``softmax``,
  ``softmax_topk``, ``topk``, ``normalizer``, and the V-split record
  functions), stream-ordered on torch's current stream.

There is no CPU fallback: every call goes through ``libosmx_b200.so``.
"""
from __future__ import annotations

import ctypes as C
from typing import NamedTuple

import numpy as np

from . import _lib
from ._lib import load

# ------------------------------------------------------------------ errors --


class OsmxError(Exception):
    """Base of the non-argument failures (CUDA errors, unsupported k)."""


class EmptyInputError(ValueError):
    """empty_input_error (error.hpp:8-10)."""

    def __init__(self, msg: str = "empty input vector"):
        super().__init__(msg)


class NonFiniteError(ValueError):
    """non_finite_error (error.hpp:13-15).  ``row`` is the first bad row."""

    def __init__(self, msg: str = "non-finite input element", row: int = -1):
        super().__init__(msg)
        self.row = row


class InvalidKError(ValueError):
    """invalid_k_error (error.hpp:18-20): k outside [1, V]."""

    def __init__(self, msg: str = "k must satisfy 1 <= k <= input size"):
        super().__init__(msg)


class InvalidChunkError(ValueError):
    """invalid_chunk_error (error.hpp:23-25)."""

    def __init__(self, msg: str = "chunk length must be >= 1"):
        super().__init__(msg)


class CudaError(OsmxError):
    pass


class NcclError(OsmxError):
    """NCCL is missing or an NCCL call of the V-split failed."""


class UnsupportedError(OsmxError):
    pass


def _raise(status: int, row: int = -1) -> None:
    if status == _lib.OK:
        return
    if status == _lib.ERR_EMPTY:
        raise EmptyInputError()
    if status == _lib.ERR_NON_FINITE:
        raise NonFiniteError(row=row)
    if status == _lib.ERR_INVALID_K:
        raise InvalidKError()
    if status == _lib.ERR_INVALID_CHUNK:
        raise InvalidChunkError()
    if status == _lib.ERR_CUDA:
        raise CudaError(load().osmx_last_cuda_error().decode())
    if status == _lib.ERR_UNSUPPORTED:
        raise UnsupportedError(f"unsupported on the device path (records need k <= {_lib.MAX_K}; "
                               "large-k top-K needs rows * k < 2^31)")
    if status == _lib.ERR_NCCL:
        raise NcclError(load().osmx_last_nccl_error().decode())
    raise ValueError(_lib.status_string(status))


class TopkResult(NamedTuple):
    """topk_result (topk.hpp:14-17): values sorted non-increasing, int64 indices."""

    values: np.ndarray
    indices: np.ndarray


class NormState(NamedTuple):
    """norm_state (normalizer.hpp:24-46): (max, sum of e^(x - max))."""

    max: float
    sum: float


ALGS = {
    "naive": _lib.NAIVE_SOFTMAX,
    "safe": _lib.SAFE_SOFTMAX,
    "online": _lib.ONLINE_SOFTMAX,
    "safe_unfused": _lib.SAFE_SOFTMAX_UNFUSED_TOPK,
    "safe_fused": _lib.SAFE_SOFTMAX_FUSED_TOPK,
    "online_fused": _lib.ONLINE_SOFTMAX_FUSED_TOPK,
    "online_unfused": _lib.ONLINE_SOFTMAX_UNFUSED_TOPK,
}

_devices: tuple[int, ...] = (0,)


def set_device(device: int) -> None:
    """CUDA device used by the host-buffer (reference-shaped) functions."""
    set_devices([device])


def set_devices(devices) -> None:
    """Devices the host-buffer functions shard a batch over: entry i takes a
    contiguous block of rows on its own host thread inside the library
    (osmx_*_host_multi; the reference's run_batch, bench.cpp:66-96).  A
    device may be listed more than once."""
    global _devices
    ds = tuple(int(d) for d in devices)
    if not ds:
        raise ValueError("set_devices needs at least one device")
    _devices = ds


def _dev_array():
    return (C.c_int * len(_devices))(*_devices), len(_devices)


# ------------------------------------------------ reference-shaped (host) --

def _as_rows(x) -> tuple[np.ndarray, bool]:
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    if a.ndim == 1:
        return a.reshape(1, -1), True
    if a.ndim != 2:
        raise ValueError("expected a 1-D vector or a 2-D batch of rows")
    return a, False


def _softmax_host(alg: int, x) -> np.ndarray:
    a, single = _as_rows(x)
    rows, V = a.shape
    if V == 0:
        raise EmptyInputError()
    y = np.empty_like(a)
    bad = C.c_int64(-1)
    devs, n = _dev_array()
    st = load().osmx_softmax_host_multi(alg, a.ctypes.data, rows, V, y.ctypes.data, devs, n, C.byref(bad))
    _raise(st, bad.value)
    return y[0] if single else y


def _topk_host(alg: int | None, x, k: int) -> TopkResult:
    a, single = _as_rows(x)
    rows, V = a.shape
    if V == 0:
        raise EmptyInputError()
    k = int(k)
    if k < 1 or k > V:
        raise InvalidKError()
    vals = np.empty((rows, k), np.float32)
    idx = np.empty((rows, k), np.int64)
    bad = C.c_int64(-1)
    devs, n = _dev_array()
    if alg is None:
        st = load().osmx_topk_host_multi(a.ctypes.data, rows, V, k, vals.ctypes.data, idx.ctypes.data, devs, n,
                                         C.byref(bad))
    else:
        st = load().osmx_softmax_topk_host_multi(alg, a.ctypes.data, rows, V, k, vals.ctypes.data,
                                                 idx.ctypes.data, devs, n, C.byref(bad))
    _raise(st, bad.value)
    if single:
        return TopkResult(vals[0], idx[0])
    return TopkResult(vals, idx)


def naive_softmax(x) -> np.ndarray:
    """Alg. 1 (softmax.hpp:13-17): no overflow guard; Inf/NaN returned as is."""
    return _softmax_host(_lib.NAIVE_SOFTMAX, x)


def safe_softmax(x) -> np.ndarray:
    """Alg. 2 (softmax.hpp:19-22): max, normalizer, outputs."""
    return _softmax_host(_lib.SAFE_SOFTMAX, x)


def online_softmax(x) -> np.ndarray:
    """Alg. 3 (softmax.hpp:24-28): fused (max, normalizer) pass, then outputs."""
    return _softmax_host(_lib.ONLINE_SOFTMAX, x)


def topk_of(values, k: int) -> TopkResult:
    """K largest values with indices, ties to the smaller index (topk.hpp:52-54)."""
    return _topk_host(None, values, k)


def safe_softmax_then_topk(x, k: int) -> TopkResult:
    """safe_softmax then topk_of, materialising y (topk.hpp:56-58)."""
    return _topk_host(_lib.SAFE_SOFTMAX_UNFUSED_TOPK, x, k)


def safe_softmax_fused_topk(x, k: int) -> TopkResult:
    """Three passes, selection on the on-the-fly probability (topk.hpp:60-63)."""
    return _topk_host(_lib.SAFE_SOFTMAX_FUSED_TOPK, x, k)


def online_softmax_topk(x, k: int) -> TopkResult:
    """Alg. 4: one pass, (m, d) + top-K of the raw logits (topk.hpp:65-68)."""
    return _topk_host(_lib.ONLINE_SOFTMAX_FUSED_TOPK, x, k)


def online_softmax_then_topk(x, k: int) -> TopkResult:
    """online_softmax then topk_of: the unfused comparator of the north star."""
    return _topk_host(_lib.ONLINE_SOFTMAX_UNFUSED_TOPK, x, k)


def _normalizer_host(x, chunk: int, precision: int):
    a, single = _as_rows(x)
    rows, V = a.shape
    if V == 0:
        raise EmptyInputError()
    dt = np.float64 if precision == 64 else np.float32
    m = np.empty(rows, dt)
    d = np.empty(rows, dt)
    bad = C.c_int64(-1)
    devs, n = _dev_array()
    st = load().osmx_normalizer_host(a.ctypes.data, rows, V, int(chunk), precision, m.ctypes.data, d.ctypes.data,
                                     devs, n, C.byref(bad))
    _raise(st, bad.value)
    if single:
        return NormState(float(m[0]), float(d[0]))
    return m, d


def run_normalizer(x, precision: int = 64):
    """(max, sum e^(x-max)) of the vector (normalizer.hpp:60-67): the state is
    double (run_normalizer<double>, the precision of the reference's kernels)
    or float (precision=32, run_normalizer<float>)."""
    return _normalizer_host(x, 0, precision)


def run_normalizer_chunked(x, chunk_len: int, precision: int = 64):
    """Chunked normalizer (normalizer.hpp:69-85): one state per contiguous
    chunk of chunk_len elements, merged left to right.  chunk_len == 0 raises
    InvalidChunkError like the reference (after the empty check)."""
    a, _ = _as_rows(x)
    if a.shape[1] == 0:
        raise EmptyInputError()
    if int(chunk_len) <= 0:
        raise InvalidChunkError()
    return _normalizer_host(x, int(chunk_len), precision)


# ---------------------------------------------------- batched (device) -----

class _Workspace:
    """Grow-only workspaces keyed by (device, stream): launches on different
    streams never share split records or a status header.  A buffer is
    allocated while its stream is current, so the caching allocator only
    reuses it in that stream's order after a regrow.  A call that skipped
    its status check (check=False) leaves the header `dirty`; the next call
    on that workspace clears it first, so a stale flag is never reported
    against other data."""

    def __init__(self):
        self.buf = {}
        self.dirty = set()

    def get(self, nbytes: int, device, stream_ptr: int):
        import torch

        key = (device.index if device.index is not None else 0, int(stream_ptr))
        t = self.buf.get(key)
        if t is None or t.numel() < nbytes:
            t = torch.zeros(max(int(nbytes), 256), dtype=torch.uint8, device=device)
            self.buf[key] = t
            self.dirty.discard(key)
        elif key in self.dirty:
            st = load().osmx_workspace_init(t.data_ptr(), t.numel(), stream_ptr)
            _raise(st)
            self.dirty.discard(key)
        return t

    def mark_dirty(self, device, stream_ptr: int):
        self.dirty.add((device.index if device.index is not None else 0, int(stream_ptr)))


_ws = _Workspace()


def _stream_ptr(device) -> int:
    import torch

    return torch.cuda.current_stream(device).cuda_stream


def _check_tensor(x, name="x"):
    import torch

    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor (the device path has no CPU fallback)")
    if x.dtype != torch.float32:
        raise TypeError(f"{name} must be float32")
    if x.dim() == 1:
        x = x.unsqueeze(0)
    if x.dim() == 2 and x.shape[1] == 0:
        raise EmptyInputError()
    if x.dim() != 2 or (x.stride(1) != 1 and x.shape[1] > 1):
        raise ValueError(f"{name} must be 1-D or 2-D with unit stride along V")
    return x


def _finish(ws, device, stream: int, check: bool) -> None:
    if check:
        check_status(ws, stream)
    else:
        _ws.mark_dirty(device, stream)


def _check_out(t, shape, dtype, device, name):
    import torch

    if not isinstance(t, torch.Tensor) or t.device != device or t.dtype != dtype or tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must be a {dtype} tensor of shape {tuple(shape)} on {device}")
    if t.numel() > 0 and (t.stride(-1) != 1 or (t.dim() == 2 and t.shape[0] > 1 and t.stride(0) < t.shape[1])):
        raise ValueError(f"{name} must have unit stride along its last dimension and non-overlapping rows")


def check_status(ws, stream: int) -> None:
    bad = C.c_int64(-1)
    st = load().osmx_check_status(ws.data_ptr(), stream, C.byref(bad))
    _raise(st, bad.value)


def workspace(alg: int, rows: int, V: int, k: int, device):
    nb = load().osmx_workspace_bytes(alg, rows, V, k)
    return _ws.get(nb, device, _stream_ptr(device)), nb


def softmax(x, alg: str = "online", out=None, check: bool = True):
    """Batched softmax of every row of a CUDA float32 tensor (rows x V)."""
    import torch

    x2 = _check_tensor(x)
    rows, V = x2.shape
    if V == 0:
        raise EmptyInputError()
    a = ALGS[alg]
    if out is None:
        out = torch.empty_like(x2)
    _check_out(out, x.shape, torch.float32, x2.device, "out")
    y = out if out.dim() == 2 else out.unsqueeze(0)
    stream = _stream_ptr(x2.device)
    ws, nb = workspace(a, rows, V, 0, x2.device)
    st = load().osmx_softmax(a, x2.data_ptr(), x2.stride(0), y.data_ptr(), y.stride(0), rows, V, ws.data_ptr(),
                             ws.numel(), stream)
    _raise(st)
    _finish(ws, x2.device, stream, check)
    return out if x.dim() == 2 else y[0]


def softmax_topk(x, k: int, alg: str = "online_fused", check: bool = True, out=None):
    """Batched softmax + top-K: returns (values rows x k, int64 indices rows x k)."""
    import torch

    x2 = _check_tensor(x)
    rows, V = x2.shape
    if V == 0:
        raise EmptyInputError()
    a = ALGS[alg]
    if out is None:
        vals = torch.empty((rows, max(k, 1)), dtype=torch.float32, device=x2.device)
        idx = torch.empty((rows, max(k, 1)), dtype=torch.int64, device=x2.device)
    else:
        vals, idx = out
        _check_out(vals, (rows, k), torch.float32, x2.device, "out[0] (values)")
        _check_out(idx, (rows, k), torch.int64, x2.device, "out[1] (indices)")
    stream = _stream_ptr(x2.device)
    ws, nb = workspace(a, rows, V, k, x2.device)
    st = load().osmx_softmax_topk(a, x2.data_ptr(), x2.stride(0), rows, V, k, vals.data_ptr(), idx.data_ptr(),
                                  ws.data_ptr(), ws.numel(), stream)
    _raise(st)
    _finish(ws, x2.device, stream, check)
    if x.dim() == 1:
        return vals[0], idx[0]
    return vals, idx


def proj_softmax_topk(h, w, k: int, check: bool = True):
    """Top-k of softmax(h @ w.T) per row without materialising the logits
    (osmx_proj_softmax_topk: tcgen05 GEMM tiles reduced to (m, d, top-k)
    records in the epilogue).  h: rows x D, w: V x D, both CUDA bfloat16,
    row-major, D % 8 == 0.  Returns (values rows x k, int64 indices)."""
    import torch

    if h.dtype != torch.bfloat16 or w.dtype != torch.bfloat16 or not (h.is_cuda and w.is_cuda):
        raise TypeError("proj_softmax_topk takes CUDA bfloat16 h and w")
    if h.dim() != 2 or w.dim() != 2 or h.shape[1] != w.shape[1]:
        raise ValueError("h must be rows x D and w V x D")
    h = h.contiguous()
    w = w.contiguous()
    rows, D = h.shape
    V = w.shape[0]
    vals = torch.empty((rows, max(k, 1)), dtype=torch.float32, device=h.device)
    idx = torch.empty((rows, max(k, 1)), dtype=torch.int64, device=h.device)
    stream = _stream_ptr(h.device)
    ws, nb = workspace(10, rows, V, k, h.device)
    st = load().osmx_proj_softmax_topk(h.data_ptr(), rows, D, w.data_ptr(), V, k, vals.data_ptr(), idx.data_ptr(),
                                       ws.data_ptr(), ws.numel(), stream)
    _raise(st)
    _finish(ws, h.device, stream, check)
    return vals, idx


def topk(v, k: int, check: bool = True):
    """Batched topk_of over a CUDA float32 tensor of values."""
    import torch

    v2 = _check_tensor(v, "v")
    rows, V = v2.shape
    if V == 0:
        raise EmptyInputError()
    vals = torch.empty((rows, max(k, 1)), dtype=torch.float32, device=v2.device)
    idx = torch.empty((rows, max(k, 1)), dtype=torch.int64, device=v2.device)
    stream = _stream_ptr(v2.device)
    ws, nb = workspace(7, rows, V, k, v2.device)
    st = load().osmx_topk(v2.data_ptr(), v2.stride(0), rows, V, k, vals.data_ptr(), idx.data_ptr(), ws.data_ptr(),
                          ws.numel(), stream)
    _raise(st)
    _finish(ws, v2.device, stream, check)
    if v.dim() == 1:
        return vals[0], idx[0]
    return vals, idx


def normalizer(x, chunk: int = 0, check: bool = True, precision: int = 32):
    """Batched (m, d) per row: float32 (precision 32) or float64 (64) tensors.
    chunk > 0: one state per contiguous chunk, merged left to right."""
    import torch

    x2 = _check_tensor(x)
    rows, V = x2.shape
    if V == 0:
        raise EmptyInputError()
    if precision not in (32, 64):
        raise ValueError("precision must be 32 or 64")
    dt = torch.float64 if precision == 64 else torch.float32
    m = torch.empty(rows, dtype=dt, device=x2.device)
    d = torch.empty(rows, dtype=dt, device=x2.device)
    stream = _stream_ptr(x2.device)
    nb = load().osmx_normalizer_workspace_bytes(rows, V, int(chunk), precision)
    ws = _ws.get(nb, x2.device, stream)
    fn = load().osmx_normalizer_f64 if precision == 64 else load().osmx_normalizer
    st = fn(x2.data_ptr(), x2.stride(0), rows, V, chunk, m.data_ptr(), d.data_ptr(), ws.data_ptr(), ws.numel(),
            stream)
    _raise(st)
    _finish(ws, x2.device, stream, check)
    return m, d


# ------------------------------------------------ V-split records (dist) ---

def record_bytes(k: int) -> int:
    return int(load().osmx_record_bytes(k))


def slice_record(x_slice, col0: int, k: int):
    """Record (m, d, top-k with global indices) of one row slice (uint8 tensor)."""
    import torch

    x1 = _check_tensor(x_slice)
    if x1.shape[0] != 1:
        raise ValueError("slice_record takes one row slice")
    V = x1.shape[1]
    rec = torch.empty(record_bytes(k), dtype=torch.uint8, device=x1.device)
    stream = _stream_ptr(x1.device)
    nb = load().osmx_workspace_bytes(9, 1, V, max(k, 1))
    ws = _ws.get(nb, x1.device, stream)
    st = load().osmx_slice_record(x1.data_ptr(), V, col0, k, rec.data_ptr(), ws.data_ptr(), ws.numel(), stream)
    _raise(st)
    _ws.mark_dirty(x1.device, stream)  # non-finite slices poison the record; its flag is not checked here
    return rec


def records_combine(records, k: int, check: bool = True):
    """Merge n records (n x record_bytes uint8 tensor, rank order).
    Returns (vals[k], idx[k], merged_record)."""
    import torch

    n = records.shape[0]
    out_rec = torch.empty(record_bytes(k), dtype=torch.uint8, device=records.device)
    vals = torch.empty(max(k, 1), dtype=torch.float32, device=records.device)
    idx = torch.empty(max(k, 1), dtype=torch.int64, device=records.device)
    stream = _stream_ptr(records.device)
    ws = _ws.get(load().osmx_workspace_bytes(0, 0, 0, 0), records.device, stream)  # the status header
    st = load().osmx_records_combine(records.data_ptr(), n, k, out_rec.data_ptr(),
                                     vals.data_ptr() if k > 0 else None, idx.data_ptr() if k > 0 else None,
                                     ws.data_ptr(), ws.numel(), stream)
    _raise(st)
    _finish(ws, records.device, stream, check)
    return vals[:k], idx[:k], out_rec


def scale_with_record(x_slice, record, out=None):
    """y = e^(x - M)/D over a slice with (M, D) from a merged record."""
    import torch

    x1 = _check_tensor(x_slice)
    if out is None:
        out = torch.empty_like(x1)
    st = load().osmx_scale_with_record(x1.data_ptr(), x1.shape[1], record.data_ptr(), out.data_ptr(),
                                       _stream_ptr(x1.device))
    _raise(st)
    return out


# ---------------------------------------------- V-split over NCCL (C-ABI) ---

class NcclComm:
    """An NCCL communicator for the C-ABI V-split (osmx_vsplit_*).  Made from
    a 128-byte unique id that rank 0 creates and the caller distributes
    (``NcclComm.from_torch_distributed`` broadcasts it over the default
    torch.distributed group).  The current CUDA device must be this rank's."""

    def __init__(self, world: int, rank: int, uid: bytes):
        import ctypes as C

        if len(uid) != 128:
            raise ValueError("an NCCL unique id is 128 bytes")
        self.world, self.rank = int(world), int(rank)
        buf = C.create_string_buffer(bytes(uid), 128)
        ptr = C.c_void_p()
        _raise(load().osmx_nccl_comm_init(C.byref(ptr), self.world, buf, self.rank))
        self.ptr = ptr.value

    @staticmethod
    def unique_id() -> bytes:
        import ctypes as C

        buf = C.create_string_buffer(128)
        _raise(load().osmx_nccl_get_unique_id(buf))
        return buf.raw

    @classmethod
    def from_torch_distributed(cls, group=None):
        import torch
        import torch.distributed as dist

        world, rank = dist.get_world_size(group), dist.get_rank(group)
        obj = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        torch.cuda.current_device()
        return cls(world, rank, obj[0])

    def close(self):
        if self.ptr:
            _raise(load().osmx_nccl_comm_destroy(self.ptr))
            self.ptr = None


def nccl_available() -> bool:
    return bool(load().osmx_nccl_available())


def vsplit_softmax_topk_nccl(x_slice, col0: int, k: int, comm: NcclComm, check: bool = True):
    """online_softmax_topk of a row split over the ranks of ``comm``: this
    rank holds columns [col0, col0 + n).  One C-ABI call: slice record ->
    ncclAllGather -> rank-order merge, all on the current stream.  Every rank
    returns the same (vals[k], idx[k]) with global column indices."""
    import torch

    if x_slice.dim() == 2:
        x_slice = x_slice.reshape(-1)
    n = int(x_slice.shape[0])
    if n and (x_slice.dtype != torch.float32 or not x_slice.is_cuda or x_slice.stride(0) != 1):
        raise ValueError("x_slice must be a contiguous float32 CUDA vector")
    dev = x_slice.device
    vals = torch.empty(k, dtype=torch.float32, device=dev)
    idx = torch.empty(k, dtype=torch.int64, device=dev)
    stream = _stream_ptr(dev)
    ws = _ws.get(load().osmx_vsplit_workspace_bytes(n, k, comm.world), dev, stream)
    st = load().osmx_vsplit_softmax_topk(x_slice.data_ptr() if n else None, n, int(col0), int(k), comm.ptr,
                                         vals.data_ptr(), idx.data_ptr(), ws.data_ptr(), ws.numel(), stream)
    _raise(st)
    _finish(ws, dev, stream, check)
    return vals, idx


def vsplit_softmax_nccl(x_slice, col0: int, comm: NcclComm, check: bool = True):
    """online_softmax of a row split over the ranks of ``comm``: returns this
    rank's slice of the probabilities."""
    import torch

    if x_slice.dim() == 2:
        x_slice = x_slice.reshape(-1)
    n = int(x_slice.shape[0])
    if n and (x_slice.dtype != torch.float32 or not x_slice.is_cuda or x_slice.stride(0) != 1):
        raise ValueError("x_slice must be a contiguous float32 CUDA vector")
    dev = x_slice.device
    y = torch.empty_like(x_slice)
    stream = _stream_ptr(dev)
    ws = _ws.get(load().osmx_vsplit_workspace_bytes(n, 0, comm.world), dev, stream)
    st = load().osmx_vsplit_softmax(x_slice.data_ptr() if n else None, n, int(col0),
                                    y.data_ptr() if n else None, comm.ptr, ws.data_ptr(), ws.numel(), stream)
    _raise(st)
    _finish(ws, dev, stream, check)
    return y
