"""Rows masked with -FLT_MAX (torch.finfo(float32).min, the usual mask value)
are finite input: the reference's double norm_state handles them
(normalizer.hpp:32-41), so every kernel family must too -- no NaN d, no
non_finite_error (the log2-domain normalizer overflowed for
maxima below -2^127)."""
from __future__ import annotations

import numpy as np
import pytest

from tests._util import max_rel

pytestmark = pytest.mark.gpu

FMIN = np.float32(np.finfo(np.float32).min)
SHAPES = {"auto": 0, "resident": 1, "stream": 2, "split": 3, "staged": 4, "cluster": 5}


@pytest.fixture
def lib():
    from paper_1805_02867_b200 import _lib

    _lib.load()
    yield _lib
    for key, val in (("shape", 0), ("split_chunk", 0), ("split_cta", -1)):
        _lib.config_set(key, val)


def masked_rows(rng, V):
    x = rng.standard_normal((10, V)).astype(np.float32)
    x[0, :] = FMIN                      # fully masked row
    x[1, : V // 2] = FMIN               # masked head, live tail
    x[2, V // 2:] = FMIN                # live head, masked tail
    x[3, ::3] = FMIN                    # strided mask
    x[4, :] = FMIN
    x[4, V - 1] = -3.0                  # one live element at the very end
    x[5, :] = -1.5e38                   # below -2^127 but not FLT_MAX
    # large magnitudes: ulp(x * log2 e) >> 1 (the log2-domain reference n
    # would be off by more than 2^7)
    x[6, :] = np.float32(3e9) + np.float32(256) * rng.integers(-3, 2, V).astype(np.float32)
    x[7, :] = (rng.standard_normal(V) * 1e20).astype(np.float32)
    x[8, :] = np.float32(3e38) - np.float32(1e31) * rng.integers(0, 4, V).astype(np.float32)
    x[9, :] = rng.standard_normal(V).astype(np.float32) * 2e6
    return x


@pytest.mark.parametrize("shape", list(SHAPES))
@pytest.mark.parametrize("V", [37, 2048, 9000, 70001])
def test_masked_softmax(cuda, oracle_mod, lib, shape, V):
    import torch

    from paper_1805_02867_b200 import osmx

    lib.config_set("shape", SHAPES[shape])
    x = masked_rows(np.random.default_rng(V), V)
    xd = torch.from_numpy(x).cuda()
    for alg in ("safe", "online"):
        y = osmx.softmax(xd, alg=alg).cpu().numpy()
        ry, st = oracle_mod.batch(f"{alg}_softmax", x)
        assert (st == 0).all()
        assert np.isfinite(y).all(), (alg, shape)
        assert max_rel(y, ry) <= 1e-5, (alg, shape)
    m, d = osmx.normalizer(xd)
    m, d = m.cpu().numpy(), d.cpu().numpy()
    for r in range(x.shape[0]):
        rm, rd, st = oracle_mod.normalizer(x[r])
        assert st == 0 and m[r] == np.float32(rm)
        assert abs(d[r] - rd) <= 1e-5 * rd, (r, d[r], rd)


@pytest.mark.parametrize("variant", [[], [("shape", 3)], [("shape", 3), ("split_cta", 0)], [("shape", 3), ("split_cta", 3)],
                                     [("shape", 3), ("split_chunk", 2048), ("split_cta", 1)]])
@pytest.mark.parametrize("V", [37, 9000, 70001])
def test_masked_fused_topk(cuda, oracle_mod, lib, variant, V):
    import torch

    from paper_1805_02867_b200 import osmx

    for key, val in variant:
        lib.config_set(key, val)
    x = masked_rows(np.random.default_rng(V + 1), V)
    vals, idx = osmx.softmax_topk(torch.from_numpy(x).cuda(), 5)
    rv, rz, st = oracle_mod.batch("online_softmax_topk", x, k=5)
    assert (st == 0).all()
    assert np.array_equal(idx.cpu().numpy(), rz)
    assert max_rel(vals.cpu().numpy(), rv) <= 1e-5
