"""GPU parity of the one-row split paths (configs[4] and the V-split slice
records): the TMA ring over dynamically claimed chunks (split_cta = 4) in
every ring layout (tma_cfg 0-2), next to the static-piece paths, for fused
online softmax + top-K (kernels.hpp:108-125) and topk_of (kernels.hpp:72-83).

Indices bit-exact against the oracle (ties to the lowest index, topk.hpp:37-43),
values within 1e-5; unaligned row starts exercise the scalar head / tail,
which only CTA 0 reads (first / last) whatever chunks it claims.  Repeated
calls check that the last CTA resets the chunk counter and the ticket.
"""
from __future__ import annotations

import numpy as np
import pytest

from tests._util import dist, max_rel

pytestmark = pytest.mark.gpu

TOL = 1e-5
PATHS = {
    "auto": [],
    "auto_split": [("shape", 3)],
    "tma0": [("shape", 3), ("split_cta", 2), ("tma_cfg", 0)],
    "dyn0": [("shape", 3), ("split_cta", 4), ("tma_cfg", 0)],
    "dyn1": [("shape", 3), ("split_cta", 4), ("tma_cfg", 1)],
    "dyn2": [("shape", 3), ("split_cta", 4), ("tma_cfg", 2)],
    "tma1": [("shape", 3), ("split_cta", 2), ("tma_cfg", 1)],
    "tma1_fused": [("shape", 3), ("split_cta", 2), ("tma_cfg", 1), ("split_fuse", 1)],
}


@pytest.fixture
def lib():
    from paper_1805_02867_b200 import _lib

    _lib.load()
    yield _lib
    for key, val in (("shape", 0), ("split_cta", -1), ("tma_cfg", -1), ("split_fuse", 0), ("split_chunk", 0)):
        _lib.config_set(key, val)


def _ref(oracle_mod, op, x, k):
    v, z, st = oracle_mod.batch(op, x, k=k)
    assert (st == 0).all()
    return v, z


@pytest.mark.parametrize("path", list(PATHS))
@pytest.mark.parametrize("k", [1, 5, 8, 32])
def test_one_row_fused_and_topk_of(cuda, oracle_mod, lib, path, k):
    import torch

    from paper_1805_02867_b200 import osmx

    for key, val in PATHS[path]:
        lib.config_set(key, val)
    rng = np.random.default_rng(700 + k)
    for V, off in ((37, 0), (4099, 1), (65536, 0), (100003, 3), (1 << 20, 2), ((1 << 22) + 5, 1)):
        for d in ("normal", "quantized2", "equal", "descending", "spikes"):
            if V > (1 << 20) and d not in ("normal", "quantized2"):
                continue
            x = dist(d, rng, 1, V + off)
            xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()[:, off:]  # row start off floats past alignment
            xs = np.ascontiguousarray(x[:, off:])
            rv, rz = _ref(oracle_mod, "online_softmax_topk", xs, k)
            for rep in range(2):
                vals, idx = osmx.softmax_topk(xd, k, alg="online_fused")
                assert np.array_equal(idx.cpu().numpy(), rz), (path, V, off, d, rep, idx[0, :4], rz[0, :4])
                assert max_rel(vals.cpu().numpy(), rv) <= TOL, (path, V, d)
            tv, ti = osmx.topk(xd, k)
            qv, qz = _ref(oracle_mod, "topk_of", xs, k)
            assert np.array_equal(ti.cpu().numpy(), qz), (path, V, off, d)
            assert np.array_equal(tv.cpu().numpy().view(np.int32), qv.view(np.int32))


@pytest.mark.parametrize("path", ["auto", "dyn0", "dyn1"])
def test_one_row_nonfinite(cuda, lib, path):
    """A NaN / +inf / -inf anywhere in the row (first, middle, last chunk,
    the scalar head or tail) raises NonFiniteError naming row 0."""
    import torch

    from paper_1805_02867_b200 import osmx

    for key, val in PATHS[path]:
        lib.config_set(key, val)
    V = (1 << 20) + 3
    for pos in (0, 1, 2, 5000, V // 2, V - 4, V - 1):
        for bad in (float("nan"), float("inf"), float("-inf")):
            x = torch.randn(1, V + 1, device="cuda")[:, 1:]
            x[0, pos] = bad
            with pytest.raises(osmx.NonFiniteError):
                osmx.softmax_topk(x, 5, alg="online_fused")
    x = torch.randn(1, V, device="cuda")  # clean after the flagged calls
    osmx.softmax_topk(x, 5, alg="online_fused")
