"""CPU: pin the oracle (our C restatement, oracle/osmx_oracle.c) before it is
trusted as the checker.

1. Bit-exact against the golden fixtures made from the REFERENCE itself
   (tests/golden/make_golden.py, run against oracle/_ref built from
   /root/reference/proj/src) -- works without /root/reference.
2. Bit-exact against oracle/_ref on fresh seeded inputs when that library is
   present (it is built here and travels to the GPU box).
3. The reference test suites' known answers (test_support.hpp:47-56,
   test_softmax.cpp, test_normalizer.cpp) and the SPEC.md top-K examples.
"""
from __future__ import annotations

import math
from pathlib import Path

import numpy as np
import pytest

from tests._util import DISTS, dist, quantized_uniform

GOLDEN = Path(__file__).resolve().parent / "golden" / "golden.npz"
SOFTMAX = ["naive_softmax", "safe_softmax", "online_softmax"]
TOPK = ["safe_softmax_then_topk", "safe_softmax_fused_topk", "online_softmax_topk", "topk_of"]

K_SOFTMAX123 = [0.090030573170380462, 0.24472847105479764, 0.66524095577482178]
K_NORM312 = 1.5032147244080551
K_NORM3120 = 1.553001792775919
K_ONE_PLUS_EXP_M2 = 1.1353352832366128
K_ONE_PLUS_EXP_M1 = 1.3678794411714423


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


def _cases(g):
    return sorted({k.split("/")[0] for k in g.files if "/x" in k})


def test_port_matches_reference_golden(oracle_mod, golden):
    O = oracle_mod
    names = _cases(golden)
    assert len(names) >= 10
    for n in names:
        x = golden[f"{n}/x"]
        k = int(golden[f"{n}/k"])
        for op in SOFTMAX:
            y, st = O.softmax(op, x)
            assert st == 0
            ref = golden[f"{n}/{op}"]
            assert np.array_equal(y.view(np.int32), ref.view(np.int32)) or (
                np.array_equal(np.isnan(y), np.isnan(ref)) and np.array_equal(y[~np.isnan(y)], ref[~np.isnan(ref)])
            ), (n, op)
        for op in TOPK:
            v, z, st = O.topk(op, x, k)
            assert st == 0
            assert np.array_equal(z, golden[f"{n}/{op}/indices"]), (n, op)
            assert np.array_equal(v.view(np.int32), golden[f"{n}/{op}/values"].view(np.int32)), (n, op)
        v, z, st = O.topk_sort(x, k)
        assert np.array_equal(z, golden[f"{n}/oracle_topk/indices"])
        ys, st = O.softmax_double(x)
        assert np.array_equal(ys, golden[f"{n}/oracle_softmax"])
        for prec in ("float", "double"):
            m, d, st = O.normalizer(x, dbl=prec == "double")
            assert [m, d] == list(golden[f"{n}/run_normalizer_{prec}"]), (n, prec)
            m, d, st = O.normalizer(x, dbl=prec == "double", chunk=7)
            assert [m, d] == list(golden[f"{n}/run_normalizer_chunked7_{prec}"]), (n, prec)


def test_count_model_matches_reference(oracle_mod, golden):
    for alg, v, k, lo, st in golden["count_accesses"]:
        a, b, s = oracle_mod.count_accesses(int(alg), int(v), int(k))
        assert s == 0 and (a, b) == (lo, st)
    # counting.hpp:83-86 access model
    V, K = 1000, 5
    tot = {alg: sum(oracle_mod.count_accesses(alg, V, K if alg >= 3 else 0)[:2]) for alg in range(6)}
    assert tot == {0: 3 * V, 1: 4 * V, 2: 3 * V, 3: 5 * V + 2 * K, 4: 3 * V + 2 * K, 5: V + 2 * K}


@pytest.mark.skipif(not (Path(__file__).resolve().parents[1] / "oracle/_ref/libosmx_ref.so").exists(),
                    reason="oracle/_ref not built")
def test_port_bit_exact_vs_reference_random(oracle_mod):
    O = oracle_mod
    rng = np.random.default_rng(1234)
    for V in (1, 2, 7, 64, 999, 4096, 30001):
        for d in DISTS:
            x = dist(d, rng, 3, V)
            for op in SOFTMAX:
                a, sa = O.batch(op, x)
                b, sb = O.batch(op, x, impl="ref")
                assert np.array_equal(sa, sb)
                assert np.array_equal(np.isnan(a), np.isnan(b))
                assert np.array_equal(np.nan_to_num(a, nan=0).view(np.int32), np.nan_to_num(b, nan=0).view(np.int32))
            k = min(V, 7)
            for op in TOPK:
                a = O.batch(op, x, k=k)
                b = O.batch(op, x, k=k, impl="ref")
                assert np.array_equal(a[1], b[1]) and np.array_equal(a[0].view(np.int32), b[0].view(np.int32)), (op, V, d)


def test_generate_inputs_golden(oracle_mod, golden):
    if not oracle_mod.ref_available():
        pytest.skip("oracle/_ref not built")
    assert np.array_equal(oracle_mod.generate_inputs(1, 3, 10), golden["generate_inputs/seed1_3x10"])
    assert oracle_mod.log_spaced_sizes(10, 1000000, 21) == list(golden["log_spaced_sizes/10_1e6_21"])


def test_known_answers_softmax(oracle_mod):
    """test_softmax.cpp:37-102."""
    O = oracle_mod
    for op in SOFTMAX:
        assert O.softmax(op, [0.0])[0][0] == 1.0
        for c in (0.0, 1.5, -20.0, 13.25):
            assert (O.softmax(op, [c] * 4)[0] == 0.25).all()
    assert O.softmax("safe_softmax", [-123.5])[0][0] == 1.0
    assert O.softmax("online_softmax", [87.0])[0][0] == 1.0
    assert (O.softmax("safe_softmax", [2.0] * 5)[0] == np.float32(1 / 5)).all()
    assert np.isnan(O.softmax("naive_softmax", [100.0, 100.0])[0]).all()
    for op in ("safe_softmax", "online_softmax"):
        assert (O.softmax(op, [100.0, 100.0])[0] == 0.5).all()
    ref, _ = O.softmax_double([1.0, 2.0, 3.0])
    assert np.allclose(ref, K_SOFTMAX123, rtol=1e-15, atol=0)
    y, _ = O.softmax("safe_softmax", [-87.0, 0.0])
    assert math.isclose(y[0], 1.6458114537543937e-38, rel_tol=1e-6) and y[1] == 1.0
    yo, _ = O.softmax("online_softmax", [-87.0, 0.0])
    assert yo[0] == y[0] and yo[1] == 1.0
    for bad in (float("nan"), float("inf"), float("-inf")):
        for op in SOFTMAX:
            assert O.softmax(op, [1.0, bad])[1] == O.NON_FINITE
    for op in SOFTMAX:
        assert O.batch(op, np.zeros((1, 0), np.float32))[1][0] == O.EMPTY


def test_known_answers_normalizer(oracle_mod):
    """test_normalizer.cpp:44-97, 133-149, 185-227."""
    O = oracle_mod
    m, d, st = O.normalizer([3.0, 1.0, 2.0])
    assert (m, st) == (3.0, 0) and math.isclose(d, K_NORM312, rel_tol=1e-12)
    m, d, st = O.normalizer([3.0, 1.0, 2.0, 0.0], chunk=2)
    assert m == 3.0 and math.isclose(d, K_NORM3120, rel_tol=1e-12)
    assert O.normalizer([1.0], chunk=0)[2] == O.INVALID_CHUNK
    assert O.normalizer([5.0]) [:2] == (5.0, 1.0)
    assert O.merge((1.0, 1.0), (2.0, 1.0))[0] == 2.0
    assert math.isclose(O.merge((1.0, 1.0), (2.0, 1.0))[1], K_ONE_PLUS_EXP_M1, rel_tol=1e-15)
    assert math.isclose(O.normalizer([3.0, 1.0])[1], K_ONE_PLUS_EXP_M2, rel_tol=1e-15)
    assert math.isclose(O.normalizer([1.0, 3.0])[1], K_ONE_PLUS_EXP_M2, rel_tol=1e-15)
    ident = (-math.inf, 0.0)
    assert O.merge(ident, ident) == ident  # no NaN from (-inf) - (-inf)
    assert O.merge(ident, (2.0, 3.0)) == (2.0, 3.0)
    # bounds 1 <= d <= j after every prefix
    rng = np.random.default_rng(42)
    x = quantized_uniform(rng, 300, 100.0)
    for j in range(1, 300, 37):
        m, d, _ = O.normalizer(x[:j])
        assert 1.0 <= d <= j and m == x[:j].max()


def test_known_answers_topk(oracle_mod):
    """SPEC.md:208-233, 294-295 and the signed-zero tie probe."""
    O = oracle_mod
    assert list(O.topk("topk_of", [0.1, 0.7, 0.2], 2)[1]) == [1, 2]
    assert list(O.topk("topk_of", [0.5, 0.5], 1)[1]) == [0]
    assert list(O.topk_sort([3, 1, 2], 3)[1]) == [0, 2, 1]
    assert list(O.topk_sort([1, 1, 1], 2)[1]) == [0, 1]
    for op in ("safe_softmax_then_topk", "safe_softmax_fused_topk", "online_softmax_topk"):
        v, z, _ = O.topk(op, [1, 2, 3], 2)
        assert list(z) == [2, 1] and np.allclose(v, K_SOFTMAX123[:0:-1], rtol=1e-6)
        assert list(O.topk(op, [2, 2, 1], 2)[1]) == [0, 1]
        v, z, _ = O.topk(op, [5.0], 1)
        assert v[0] == 1.0 and z[0] == 0
        assert O.topk(op, [1.0, 2.0], 3)[2] == O.INVALID_K
        assert O.topk(op, [1.0, 2.0], 0)[2] == O.INVALID_K
    assert list(O.topk("online_softmax_topk", [0, -0.0, 1, 1, -0.0, 0], 4)[1]) == [2, 3, 0, 1]


def test_cpu_batch_threads_agree(oracle_mod):
    """The row-striped multi-thread driver (bench.cpp:75-90 analogue) changes
    nothing numerically."""
    rng = np.random.default_rng(3)
    x = rng.standard_normal((33, 777)).astype(np.float32)
    a = oracle_mod.batch("online_softmax_topk", x, k=5, threads=1)
    b = oracle_mod.batch("online_softmax_topk", x, k=5, threads=4)
    assert np.array_equal(a[1], b[1]) and np.array_equal(a[0], b[0])
