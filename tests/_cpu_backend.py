"""CPU stand-in for shard.CudaBackend (TEST INFRASTRUCTURE): produces and
merges records in the library's byte layout (topk_impl.cuh RecHdr:
float m, d, mn; int k; float v[k] padded to 8 B; int64 idx[k]) with the
oracle's arithmetic, so the gloo tests exercise the real host-side exchange
and ordering logic of paper_1805_02867_b200.shard without a GPU."""
from __future__ import annotations

import math
import struct

import numpy as np
import torch

from oracle import oracle as O


def _layout(k):
    kk = max(k, 1)
    idx_off = 16 + ((4 * kk + 7) // 8) * 8
    rb = ((idx_off + 8 * kk) + 15) // 16 * 16
    return kk, idx_off, rb


class CpuBackend:
    def record_bytes(self, k):
        return _layout(k)[2]

    def _pack(self, m, d, mn, k, vals, idx):
        kk, idx_off, rb = _layout(k)
        buf = bytearray(rb)
        struct.pack_into("<fffi", buf, 0, m, d, mn, kk)
        for r in range(kk):
            struct.pack_into("<f", buf, 16 + 4 * r, vals[r] if r < len(vals) else float("-inf"))
            struct.pack_into("<q", buf, idx_off + 8 * r, int(idx[r]) if r < len(idx) else -1)
        return torch.frombuffer(buf, dtype=torch.uint8).clone()

    def _unpack(self, rec, k):
        kk, idx_off, rb = _layout(k)
        b = bytes(rec.numpy().tobytes())
        m, d, mn, _ = struct.unpack_from("<fffi", b, 0)
        vals = [struct.unpack_from("<f", b, 16 + 4 * r)[0] for r in range(kk)]
        idx = [struct.unpack_from("<q", b, idx_off + 8 * r)[0] for r in range(kk)]
        return m, d, mn, vals, idx

    def empty_record(self, k, device=None):
        kk = max(k, 1)
        return self._pack(float("-inf"), 0.0, float("inf"), k, [float("-inf")] * kk, [-1] * kk)

    def slice_record(self, x_slice, col0, k):
        x = x_slice.reshape(-1).numpy().astype(np.float32)
        m, d, _ = O.normalizer(x, dbl=True)
        kk = max(k, 1)
        n = min(kk, x.size)
        v, z, _ = O.topk_sort(x, n)
        return self._pack(m, d, float(x.min()), k, list(v), [int(i) + col0 for i in z])

    def combine(self, records, k):
        kk = max(k, 1)
        M, D = float("-inf"), 0.0
        cands = []
        for r in range(records.shape[0]):
            m, d, mn, vals, idx = self._unpack(records[r], k)
            M, D = O.merge((M, D), (m, d))  # rank (column) order, normalizer.hpp:82
            cands += [(v, i) for v, i in zip(vals, idx) if i >= 0]
        cands.sort(key=lambda t: (-t[0], t[1]))  # oracle.cpp:48-51
        top = cands[:kk]
        vals = torch.tensor([math.exp(v - M) / D for v, _ in top], dtype=torch.float32)
        idx = torch.tensor([i for _, i in top], dtype=torch.int64)
        merged = self._pack(M, D, 0.0, k, [v for v, _ in top], [i for _, i in top])
        return vals[:k], idx[:k], merged

    def scale(self, x_slice, record):
        m, d, _, _, _ = self._unpack(record, 0)
        x = x_slice.reshape(-1).double()
        return (torch.exp(x - m) / d).float().reshape(1, -1)
