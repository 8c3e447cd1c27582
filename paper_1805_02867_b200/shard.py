"""Multi-GPU row sharder and V-split combine (one process per GPU).

Two ways the north star spreads the hot path over the GPUs of one box:

* **Row sharding** (configs[3], C4): rows are independent, so rank r takes the
  contiguous block [r*N/G, (r+1)*N/G) and runs the batched kernel on it.  No
  collective touches the data path -- the CPU analogue is the reference's
  row striping over std::threads (bench.cpp:75-90).

* **V-split** (configs[4], C5: one row too long for one device): rank r takes
  the contiguous column slice [c_r, c_{r+1}), reduces it on-device to one
  record -- the paper's (m, d) state plus k (value, global index) candidates
  (Eq. 4-5; normalizer.hpp:52-58, topk.hpp:34-44) -- and ONE all-gather of the
  fixed-size records (NCCL over NVLink) gives every rank all G records, which
  it merges in rank (= column) order, exactly the reference's chunked
  normalizer (normalizer.hpp:73-85) with the chunk boundaries at the rank
  boundaries.  Softmax then rescales its own slice against the merged (M, D).

The device work goes through ``osmx`` (the C-ABI); the exchange through
``torch.distributed``.  ``backend`` is injectable so the host logic is tested
on CPU with gloo (tests/test_dist.py).
"""
from __future__ import annotations

from dataclasses import dataclass


def row_range(rows: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row block of `rank` (sizes differ by at most one row)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, rem = divmod(rows, world)
    r0 = rank * base + min(rank, rem)
    return r0, r0 + base + (1 if rank < rem else 0)


def col_range(V: int, world: int, rank: int, align: int = 16) -> tuple[int, int]:
    """Contiguous column slice of `rank`.  Boundaries are multiples of `align`
    elements (64 bytes) so every slice keeps the row's 16-byte phase; the last
    rank takes the remainder.  Slices may be empty when V < world*align."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    per = -(-V // world)
    per = -(-per // align) * align
    c0 = min(V, rank * per)
    return c0, min(V, c0 + per)


@dataclass
class CudaBackend:
    """Device operations of the V-split, all through the C-ABI."""

    def slice_record(self, x_slice, col0: int, k: int):
        from . import osmx

        return osmx.slice_record(x_slice, col0, k)

    def record_bytes(self, k: int) -> int:
        from . import osmx

        return osmx.record_bytes(k)

    def combine(self, records, k: int):
        from . import osmx

        return osmx.records_combine(records, k)

    def scale(self, x_slice, record):
        from . import osmx

        return osmx.scale_with_record(x_slice, record)

    def empty_record(self, k: int, device):
        """Record of an empty slice: the merge identity (-inf, 0), no candidates."""
        import struct

        import torch

        rb = self.record_bytes(k)
        kk = max(k, 1)
        hdr = struct.pack("<fffi", float("-inf"), 0.0, float("inf"), kk)
        vals_off = 16
        idx_off = 16 + ((4 * kk + 7) // 8) * 8
        buf = bytearray(rb)
        buf[0:16] = hdr
        for r in range(kk):
            struct.pack_into("<f", buf, vals_off + 4 * r, float("-inf"))
            struct.pack_into("<q", buf, idx_off + 8 * r, -1)
        return torch.frombuffer(buf, dtype=torch.uint8).to(device)


def _all_gather_records(rec, world: int, group=None):
    import torch
    import torch.distributed as dist

    out = torch.empty((world, rec.numel()), dtype=rec.dtype, device=rec.device)
    try:
        dist.all_gather_into_tensor(out.view(-1), rec.contiguous(), group=group)
    except (RuntimeError, NotImplementedError):  # backends without the fused form (gloo)
        parts = list(out.unbind(0))
        dist.all_gather(parts, rec.contiguous(), group=group)
    return out


def vsplit_softmax_topk(x_slice, col0: int, k: int, world: int, group=None, backend=None):
    """Top-k (values, global indices) of one row split over `world` ranks.
    x_slice: this rank's columns (1 x n, may be n == 0).  Every rank returns
    the same result."""
    be = backend or CudaBackend()
    if x_slice.shape[-1] == 0:
        rec = be.empty_record(k, x_slice.device)
    else:
        rec = be.slice_record(x_slice.reshape(1, -1), col0, k)
    recs = _all_gather_records(rec, world, group)
    vals, idx, _ = be.combine(recs, k)
    return vals, idx


def vsplit_softmax(x_slice, col0: int, world: int, group=None, backend=None):
    """Softmax of one row split over `world` ranks: each rank returns its own
    slice of the probabilities."""
    be = backend or CudaBackend()
    if x_slice.shape[-1] == 0:
        rec = be.empty_record(0, x_slice.device)
    else:
        rec = be.slice_record(x_slice.reshape(1, -1), col0, 0)
    recs = _all_gather_records(rec, world, group)
    _, _, merged = be.combine(recs, 0)
    if x_slice.shape[-1] == 0:
        return x_slice.clone()
    return be.scale(x_slice.reshape(1, -1), merged)


def sharded_rows(x_full_rows: int, world: int, rank: int):
    """Row block helper used by bench.py and the tests."""
    return row_range(x_full_rows, world, rank)
