"""The host-buffer row sharder (osmx_*_host_multi; the reference's run_batch
stripes rows over std::threads, bench.cpp:66-96), per-call launch knobs
(reentrancy, softmax.hpp:8-9) and the workspace rules of the Python layer.

A device may be listed twice, so the multi-thread / multi-context paths run
on a one-GPU box: [0, 0] drives device 0 from two host threads with two
staging contexts."""
from __future__ import annotations

import ctypes as C
import threading

import numpy as np
import pytest

from tests._util import dist, max_rel

pytestmark = pytest.mark.gpu


@pytest.fixture
def lib():
    from paper_1805_02867_b200 import _lib, osmx

    _lib.load()
    yield _lib
    osmx.set_devices([0])
    for key, val in (("shape", 0), ("split_chunk", 0), ("host_chunk_mb", 512), ("split_cta", -1)):
        _lib.config_set(key, val)


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0]])
@pytest.mark.parametrize("alg,op", [("online_fused", "online_softmax_topk"),
                                    ("safe_fused", "safe_softmax_fused_topk")])
def test_multi_device_topk_bit_exact(cuda, oracle_mod, lib, devices, alg, op):
    from paper_1805_02867_b200 import osmx

    rng = np.random.default_rng(11)
    x = dist("quantized2", rng, 97, 5003)  # dense ties: index order matters
    osmx.set_devices(devices)
    fn = {"online_fused": osmx.online_softmax_topk, "safe_fused": osmx.safe_softmax_fused_topk}[alg]
    got = fn(x, 5)
    rv, rz, st = oracle_mod.batch(op, x, k=5)
    assert (st == 0).all()
    assert np.array_equal(got.indices, rz)
    assert max_rel(got.values, rv) <= 1e-5


@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0, 0]])
def test_multi_device_softmax_and_topk_of(cuda, oracle_mod, lib, devices):
    from paper_1805_02867_b200 import osmx

    rng = np.random.default_rng(12)
    x = dist("normal", rng, 33, 3001)
    osmx.set_devices(devices)
    y = osmx.online_softmax(x)
    ry, st = oracle_mod.batch("online_softmax", x)
    assert max_rel(y, ry) <= 1e-5
    t = osmx.topk_of(x, 7)
    rv, rz, _ = oracle_mod.batch("topk_of", x, k=7)
    assert np.array_equal(t.indices, rz) and np.array_equal(t.values, rv)


def test_multi_device_first_bad_row_is_global(cuda, lib):
    """A non-finite row in the second device's block is reported with its
    global row index."""
    from paper_1805_02867_b200 import osmx

    x = np.random.default_rng(13).standard_normal((40, 1000)).astype(np.float32)
    x[31, 500] = np.nan
    x[37, 2] = np.inf
    osmx.set_devices([0, 0])
    with pytest.raises(osmx.NonFiniteError) as e:
        osmx.online_softmax_topk(x, 5)
    assert e.value.row == 31


def test_multi_device_rejects_bad_device(cuda, lib):
    lib_ = lib.load()
    x = np.zeros((4, 16), np.float32)
    v = np.empty((4, 2), np.float32)
    i = np.empty((4, 2), np.int64)
    devs = (C.c_int * 2)(0, 4096)
    bad = C.c_int64(0)
    st = lib_.osmx_softmax_topk_host_multi(5, x.ctypes.data, 4, 16, 2, v.ctypes.data, i.ctypes.data, devs, 2,
                                           C.byref(bad))
    assert st == lib.ERR_INVALID_ARG
    st = lib_.osmx_softmax_topk_host_multi(5, x.ctypes.data, 4, 16, 2, v.ctypes.data, i.ctypes.data, devs, 0,
                                           C.byref(bad))
    assert st == lib.ERR_INVALID_ARG


def test_host_tail_block_takes_split_path(cuda, oracle_mod, lib):
    """the short tail block of the host pipeline may pick the
    split-record shape when the full blocks did not; its workspace must be
    sized for it.  1 MB blocks of V=100000 rows = 2 rows per block, so 5
    rows leave a 1-row tail (split path: rows < 5 x SMs and V > 65536 for
    every block here, and the softmax split for the tail)."""
    from paper_1805_02867_b200 import osmx

    lib.config_set("host_chunk_mb", 1)
    rng = np.random.default_rng(14)
    x = dist("normal", rng, 5, 100000)
    got = osmx.online_softmax_topk(x, 5)
    rv, rz, _ = oracle_mod.batch("online_softmax_topk", x, k=5)
    assert np.array_equal(got.indices, rz)
    y = osmx.online_softmax(x)
    ry, _ = oracle_mod.batch("online_softmax", x)
    assert max_rel(y, ry) <= 1e-5
    # 1400 rows x 100000 with 512 MB blocks: 1342-row blocks + a 58-row tail
    lib.config_set("host_chunk_mb", 512)
    x = dist("normal", rng, 1400, 100000)
    got = osmx.online_softmax_topk(x, 5)
    rv, rz, _ = oracle_mod.batch("online_softmax_topk", x, k=5)
    assert np.array_equal(got.indices, rz)


def test_concurrent_slice_record_does_not_leak_shape(cuda, oracle_mod, lib):
    """osmx_slice_record forces the split shape for its own call only: a
    concurrent osmx_softmax_topk on another thread keeps the default shape
    and stays bit-exact, and the process default is unchanged afterwards."""
    import torch

    from paper_1805_02867_b200 import osmx

    rng = np.random.default_rng(15)
    xr = dist("normal", rng, 1, 300000)
    xs = dist("quantized2", rng, 64, 4099)
    rv, rz, _ = oracle_mod.batch("online_softmax_topk", xs, k=5)
    errors = []
    stop = threading.Event()

    def recorder():
        try:
            dev = torch.device("cuda", 0)
            s = torch.cuda.Stream(dev)
            with torch.cuda.stream(s):
                xd = torch.from_numpy(xr).to(dev)
                while not stop.is_set():
                    osmx.slice_record(xd, 0, 5)
                s.synchronize()
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    th = threading.Thread(target=recorder)
    th.start()
    try:
        xd = torch.from_numpy(xs).cuda()
        for _ in range(50):
            vals, idx = osmx.softmax_topk(xd, 5)
            assert np.array_equal(idx.cpu().numpy(), rz)
    finally:
        stop.set()
        th.join()
    assert not errors, errors
    assert lib.config_get("shape") == 0


def test_unchecked_call_does_not_poison_next_checked_call(cuda, lib):
    """a check=False call on a bad row must not make the next
    checked call on clean data raise with a stale row index."""
    import torch

    from paper_1805_02867_b200 import osmx

    bad = torch.randn(8, 1000, device="cuda")
    bad[3, 10] = float("nan")
    osmx.softmax_topk(bad, 5, check=False)
    good = torch.randn(8, 1000, device="cuda")
    osmx.softmax(good)  # different op, same stream: must not raise
    osmx.softmax_topk(good, 5)
    with pytest.raises(osmx.NonFiniteError):
        osmx.softmax_topk(bad, 5)


def test_out_arguments_are_validated(cuda, lib):
    import torch

    from paper_1805_02867_b200 import osmx

    x = torch.randn(4, 100, device="cuda")
    with pytest.raises(ValueError):
        osmx.softmax(x, out=torch.empty(4, 99, device="cuda"))
    with pytest.raises(ValueError):
        osmx.softmax(x, out=torch.empty(100, 4, device="cuda").t())
    with pytest.raises(ValueError):
        osmx.softmax(x, out=torch.empty(4, 100, device="cuda", dtype=torch.float64))
    with pytest.raises(ValueError):
        osmx.softmax_topk(x, 5, out=(torch.empty(4, 5, device="cuda"), torch.empty(4, 5, device="cuda",
                                                                                       dtype=torch.int32)))
    with pytest.raises(ValueError):
        osmx.softmax_topk(x, 5, out=(torch.empty(4, 4, device="cuda"), torch.empty(4, 5, device="cuda",
                                                                                       dtype=torch.int64)))
    v, i = torch.empty(4, 5, device="cuda"), torch.empty(4, 5, device="cuda", dtype=torch.int64)
    osmx.softmax_topk(x, 5, out=(v, i))
    ref = torch.topk(torch.softmax(x, 1), 5)
    assert torch.equal(i, ref.indices)
