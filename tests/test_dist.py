"""CPU, world_size 2 (gloo): the multi-GPU host logic of
paper_1805_02867_b200.shard -- row blocks, column slices, the rank-ordered
record all-gather and merge -- against the oracle on the whole row."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1805_02867_b200.shard import col_range, row_range


def test_row_range_partition():
    for rows in (0, 1, 7, 65536, 65537):
        for world in (1, 2, 3, 8):
            spans = [row_range(rows, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == rows
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_col_range_partition():
    for V in (1, 15, 16, 100, 1 << 26, (1 << 26) + 5):
        for world in (1, 2, 4, 8):
            spans = [col_range(V, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == V
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert all(a % 16 == 0 or a == V for a, _ in spans)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, V, k, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1805_02867_b200.shard import vsplit_softmax, vsplit_softmax_topk
        from tests._cpu_backend import CpuBackend

        rng = np.random.default_rng(seed)
        x = rng.standard_normal(V).astype(np.float32)
        x[V // 3] = x[2 * V // 3] = 9.0  # an exact tie across ranks
        c0, c1 = col_range(V, world, rank)
        xs = torch.from_numpy(x[c0:c1].copy()).reshape(1, -1)
        vals, idx = vsplit_softmax_topk(xs, c0, k, world, backend=CpuBackend())
        y = vsplit_softmax(xs, c0, world, backend=CpuBackend())
        q.put((rank, c0, c1, vals.numpy(), idx.numpy(), y.numpy().reshape(-1)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("V,k", [(1000, 5), (37, 5), (20, 3)])
def test_vsplit_gloo_world2(oracle_mod, V, k):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, V, k, 7, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(7)
    x = rng.standard_normal(V).astype(np.float32)
    x[V // 3] = x[2 * V // 3] = 9.0
    rv, rz, st = oracle_mod.topk("online_softmax_topk", x, k)
    ry, _ = oracle_mod.softmax("online_softmax", x)
    y = np.zeros(V, np.float32)
    for rank, c0, c1, vals, idx, ys in res:
        assert np.array_equal(idx, rz), (rank, idx, rz)  # same answer on every rank
        assert np.allclose(vals, rv, rtol=1e-6)
        y[c0:c1] = ys
    assert np.allclose(y, ry, rtol=1e-6, atol=0)


def _gpu_worker(rank, world, port, V, k, seed, q):
    """Both ranks on cuda:0: the real CUDA records (osmx_slice_record /
    osmx_records_combine / osmx_scale_with_record) exchanged over gloo."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1805_02867_b200.shard import vsplit_softmax, vsplit_softmax_topk

        rng = np.random.default_rng(seed)
        x = rng.standard_normal(V).astype(np.float32)
        c0, c1 = col_range(V, world, rank)
        xs = torch.from_numpy(x[c0:c1].copy()).reshape(1, -1).cuda()
        vals, idx = vsplit_softmax_topk(xs, c0, k, world)
        y = vsplit_softmax(xs, c0, world)
        q.put((rank, c0, c1, vals.cpu().numpy(), idx.cpu().numpy(), y.cpu().numpy().reshape(-1)))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("V,k,world", [(1 << 20, 5, 2), (300001, 8, 3)])
def test_vsplit_cuda_records_multiprocess(oracle_mod, V, k, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, V, k, 11, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    x = np.random.default_rng(11).standard_normal(V).astype(np.float32)
    rv, rz, st = oracle_mod.topk("online_softmax_topk", x, k)
    ry, _ = oracle_mod.softmax("online_softmax", x)
    y = np.zeros(V, np.float32)
    for rank, c0, c1, vals, idx, ys in res:
        assert np.array_equal(idx.reshape(-1), rz), (rank, idx, rz)
        assert np.allclose(vals.reshape(-1), rv, rtol=1e-5)
        y[c0:c1] = ys
    m = ry > 1e-30
    assert np.max(np.abs(y[m].astype(np.float64) - ry[m]) / ry[m]) <= 1e-5
