"""Randomised parity over the launch space: row count, V, leading dimension
and base offset (16-byte phase), k (register lists and the large-k path),
algorithm and forced kernel family, all against the oracle."""
from __future__ import annotations

import numpy as np
import pytest

from tests._util import dist, max_rel

pytestmark = pytest.mark.gpu

SHAPES = [0, 1, 2, 3, 4, 5]
DISTS = ["normal", "quantized2", "spikes", "wide", "equal"]


@pytest.fixture
def lib():
    from paper_1805_02867_b200 import _lib

    _lib.load()
    yield _lib
    for key, val in (("shape", 0), ("split_chunk", 0), ("cluster_size", 0)):
        _lib.config_set(key, val)


def test_random_launch_space(cuda, oracle_mod, lib):
    import torch

    from paper_1805_02867_b200 import osmx

    rng = np.random.default_rng(2026)
    n_checked = 0
    for case in range(400):
        rows = int(rng.choice([1, 2, 7, 33, 150, 300]))
        V = int(rng.choice([1, 3, 17, 255, 1000, 2047, 4099, 9000, 16387, 30001, 70001]))
        if rows * V > 4_000_000:
            rows = max(1, 4_000_000 // V)
        off = int(rng.integers(0, 4))
        pad = int(rng.integers(0, 5))
        shape = int(rng.choice(SHAPES))
        if shape == 1 and V + 3 > 16384:
            shape = 0
        lib.config_set("shape", shape)
        lib.config_set("split_chunk", int(rng.choice([0, 2048, 8192])) if shape == 3 else 0)
        lib.config_set("cluster_size", int(rng.choice([0, 2, 3])) if shape == 5 else 0)
        d = str(rng.choice(DISTS))
        base = dist(d, rng, rows, V + off + pad)
        x = np.ascontiguousarray(base[:, off:off + V])
        xt = torch.from_numpy(base).cuda()[:, off:off + V]  # ld = V + off + pad, base phase = off
        kind = rng.integers(0, 3)
        ctx = (case, rows, V, off, pad, shape, d)
        if kind == 0:
            alg = str(rng.choice(["naive", "safe", "online"]))
            if alg == "naive" and d in ("wide", "spikes"):
                alg = "online"
            y = osmx.softmax(xt, alg=alg).cpu().numpy()
            ref, st = oracle_mod.batch(f"{alg}_softmax", x)
            assert max_rel(y, ref) <= 1e-5, (alg,) + ctx
        elif kind == 1:
            k = int(min(V, rng.choice([1, 5, 13, 32, 33, 100])))
            vals, idx = osmx.softmax_topk(xt, k, alg="online_fused")
            rv, rz, _ = oracle_mod.batch("online_softmax_topk", x, k=k)
            assert np.array_equal(idx.cpu().numpy(), rz), ("fused", k) + ctx
            assert max_rel(vals.cpu().numpy(), rv) <= 1e-5, ("fused", k) + ctx
        else:
            k = int(min(V, rng.choice([1, 5, 16, 40])))
            vals, idx = osmx.topk(xt, k)
            rv, rz, _ = oracle_mod.batch("topk_of", x, k=k)
            assert np.array_equal(idx.cpu().numpy(), rz), ("topk_of", k) + ctx
            assert np.array_equal(vals.cpu().numpy().view(np.int32), rv.view(np.int32)), ("topk_of", k) + ctx
        n_checked += 1
    print(f"{n_checked} random launches checked")
