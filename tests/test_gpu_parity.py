"""GPU parity: every batched entry point of the C-ABI against the oracle
(our C restatement, itself pinned bit-exactly to the reference in
test_oracle.py) on the same seeded inputs.

Bars (BASELINE.json north_star): fp32 probabilities within max relative
error 1e-5 (reference values <= 1e-30 skipped, test_softmax.cpp:30); top-K
indices bit-exact with ties to the lowest index.  Every kernel family
(resident / stream / split) is forced in turn.
"""
from __future__ import annotations

import numpy as np
import pytest

from tests._util import DISTS, dist, max_rel

pytestmark = pytest.mark.gpu

TOL = 1e-5
SHAPES = {"auto": 0, "resident": 1, "stream": 2, "split": 3, "staged": 4, "cluster": 5}
# top-K launch variants: knob settings applied on top of the shape
TOPK_VARIANTS = {
    "auto": [], "stream": [("shape", 2)], "split": [("shape", 3), ("split_chunk", 2048)], "tma": [("tma", 2)],
    "warp": [("topk_threads", 32), ("topk_u8", 0)], "warp_u8": [("topk_threads", 32), ("topk_u8", 1)],
    "warp_pf": [("topk_threads", 32), ("l2_prefetch", 2)], "cta_pf": [("topk_threads", 256), ("l2_prefetch", 1)],
    "warp_pipe1": [("topk_threads", 32), ("topk_pipe", 1)], "warp_pipe2": [("topk_threads", 32), ("topk_pipe", 2)],
    "warp_pipe3": [("topk_threads", 32), ("topk_pipe", 3)],
    "warp_db4": [("topk_threads", 32), ("topk_pipe", 4)], "warp_db2": [("topk_threads", 32), ("topk_pipe", 5)],
    "warp_bulk": [("topk_threads", 32), ("topk_pipe", 6)],
    "split_cta": [("shape", 3), ("split_chunk", 2048), ("split_cta", 1)],
    "split_auto": [("shape", 3)],
    "split_warp": [("shape", 3), ("split_chunk", 2048), ("split_cta", 0)],
    "split_warp_auto": [("shape", 3), ("split_cta", 0)],
    "split_tma": [("shape", 3), ("split_cta", 2)],
    "split_tma_small": [("shape", 3), ("split_chunk", 2048), ("split_cta", 2)],
    "split_wide": [("shape", 3), ("split_cta", 3)],
}


@pytest.fixture
def lib():
    from paper_1805_02867_b200 import _lib

    _lib.load()
    yield _lib
    for key, val in (("shape", 0), ("split_chunk", 0), ("tma", 0), ("topk_threads", 0), ("topk_u8", -1),
                     ("l2_prefetch", -1), ("cluster_size", 0), ("topk_pipe", 0), ("split_cta", -1)):
        _lib.config_set(key, val)


def _dev(x):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


SOFTMAX_V = [1, 2, 3, 5, 10, 17, 32, 33, 100, 255, 256, 1000, 1023, 1025, 2048, 4099, 8192, 16384, 16387, 70001]


@pytest.mark.parametrize("shape", ["auto", "resident", "stream", "split", "staged", "cluster"])
@pytest.mark.parametrize("alg", ["naive", "safe", "online"])
def test_softmax_parity(cuda, oracle_mod, lib, alg, shape):
    from paper_1805_02867_b200 import osmx

    lib.config_set("shape", SHAPES[shape])
    if shape == "split":
        lib.config_set("split_chunk", 4096)
    rng = np.random.default_rng(100 + SHAPES[shape])
    worst = 0.0
    for V in SOFTMAX_V:
        if shape in ("resident", "staged") and V > 16384:
            continue
        for d in DISTS:
            if alg == "naive" and d in ("wide", "spikes", "quantized100"):
                continue  # overflow regime: covered by test_naive_overflow
            rows = 3 if V > 10000 else 7
            x = dist(d, rng, rows, V)
            y = osmx.softmax(_dev(x), alg=alg).cpu().numpy()
            ref, st = oracle_mod.batch(f"{alg}_softmax", x)
            assert (st == 0).all()
            err = max_rel(y, ref)
            worst = max(worst, err)
            assert err <= TOL, f"{alg}/{shape} V={V} dist={d}: max rel err {err:.3g}"
    print(f"{alg}/{shape}: worst rel err {worst:.3g}")


@pytest.mark.parametrize("alg", ["safe", "online", "naive"])
def test_softmax_strided_and_misaligned(cuda, oracle_mod, lib, alg):
    """Leading dimension > V and a row base that is not 16-byte aligned
    exercise the head/body/tail split of every row."""
    import torch

    from paper_1805_02867_b200 import osmx

    rng = np.random.default_rng(7)
    for shape in (0, 2, 3, 4, 5):
        lib.config_set("shape", shape)
        lib.config_set("split_chunk", 4096 if shape == 3 else 0)
        lib.config_set("cluster_size", 4 if shape == 5 else 0)
        for V in (5, 999, 4097, 20001, 70003):
            big = rng.standard_normal((6, V + 7)).astype(np.float32)
            xt = torch.from_numpy(big).cuda()[:, 1 : V + 1]  # ld = V+7, base offset 4 bytes
            y = osmx.softmax(xt, alg=alg).cpu().numpy()
            ref, _ = oracle_mod.batch(f"{alg}_softmax", np.ascontiguousarray(big[:, 1 : V + 1]))
            assert max_rel(y, ref) <= TOL, (alg, shape, V)


def test_softmax_known_answers(cuda, lib):
    """test_softmax.cpp:37-102 goldens through the device path."""
    from paper_1805_02867_b200 import osmx

    def sm(a, x):
        return osmx.softmax(_dev(np.asarray(x, np.float32).reshape(1, -1)), alg=a).cpu().numpy()[0]

    for a in ("naive", "safe", "online"):
        assert sm(a, [0.0])[0] == 1.0
        for c in (0.0, 1.5, -20.0, 13.25):
            assert (sm(a, [c] * 4) == 0.25).all()
    assert sm("safe", [-123.5])[0] == 1.0
    assert sm("online", [87.0])[0] == 1.0
    assert (sm("safe", [2.0] * 5) == np.float32(1.0 / 5.0)).all()
    yn = sm("naive", [100.0, 100.0])
    assert np.isnan(yn).all()
    for a in ("safe", "online"):
        assert (sm(a, [100.0, 100.0]) == 0.5).all()
    assert not np.isfinite(sm("naive", [50.0, 89.0, 0.0])).all()
    assert np.isfinite(sm("safe", [50.0, 89.0, 0.0])).all()
    k123 = np.array([0.090030573170380462, 0.24472847105479764, 0.66524095577482178])
    for a in ("naive", "safe", "online"):
        assert max_rel(sm(a, [1.0, 2.0, 3.0]), k123) <= 1e-6
    y = sm("safe", [-87.0, 0.0])
    assert abs(y[0] - 1.6458114537543937e-38) <= 1e-6 * 1.6458114537543937e-38
    assert y[1] == 1.0
    yo = sm("online", [-87.0, 0.0])
    assert yo[0] == y[0] and yo[1] == 1.0


def test_naive_overflow_positions(cuda, oracle_mod, lib):
    """Naive has no overflow guard: non-finite output positions must match the
    reference's (kernels.hpp:39-46)."""
    from paper_1805_02867_b200 import osmx

    rng = np.random.default_rng(11)
    for V in (3, 100, 5000):
        x = (rng.uniform(80, 200, size=(4, V)) * rng.choice([-1, 1], size=(4, V))).astype(np.float32)
        y = osmx.softmax(_dev(x), alg="naive").cpu().numpy()
        ref, _ = oracle_mod.batch("naive_softmax", x)
        assert np.array_equal(np.isfinite(y), np.isfinite(ref))
        assert np.array_equal(np.isnan(y), np.isnan(ref))
        fin = np.isfinite(ref)
        assert np.allclose(y[fin], ref[fin], rtol=1e-5, atol=1e-30)


TOPK_V = [1, 2, 5, 10, 33, 100, 1000, 2049, 4099, 32768, 100003]


def _topk_ref(oracle_mod, op, x, k):
    v, z, st = oracle_mod.batch(op, x, k=k)
    assert (st == 0).all()
    return v, z


@pytest.mark.parametrize("shape", list(TOPK_VARIANTS))
@pytest.mark.parametrize("k", [1, 2, 5, 8, 13, 32])
def test_online_fused_topk_parity(cuda, oracle_mod, lib, shape, k):
    """Alg. 4: indices bit-exact (ties to the lowest index), values 1e-5."""
    from paper_1805_02867_b200 import osmx

    for key, val in TOPK_VARIANTS[shape]:
        lib.config_set(key, val)
    rng = np.random.default_rng(200 + k)
    for V in TOPK_V:
        if k > V:
            continue
        for d in DISTS:
            rows = 3 if V > 10000 else 9
            x = dist(d, rng, rows, V)
            vals, idx = osmx.softmax_topk(_dev(x), k, alg="online_fused")
            rv, rz = _topk_ref(oracle_mod, "online_softmax_topk", x, k)
            got = idx.cpu().numpy()
            assert np.array_equal(got, rz), f"V={V} k={k} {d} {shape}: {got[:2]} vs {rz[:2]}"
            assert max_rel(vals.cpu().numpy(), rv) <= TOL


@pytest.mark.parametrize("shape", ["auto", "split", "tma"])
@pytest.mark.parametrize("k", [1, 5, 16])
def test_topk_of_parity(cuda, oracle_mod, lib, shape, k):
    """topk_of: values and indices bit-exact (kernels.hpp:72-83)."""
    from paper_1805_02867_b200 import osmx

    if shape == "tma":
        lib.config_set("tma", 2)
        shape = "auto"
    else:
        lib.config_set("tma", 0)
    lib.config_set("shape", SHAPES[shape])
    if shape == "split":
        lib.config_set("split_chunk", 2048)
    rng = np.random.default_rng(300 + k)
    for V in TOPK_V:
        if k > V:
            continue
        for d in DISTS:
            x = dist(d, rng, 5, V)
            vals, idx = osmx.topk(_dev(x), k)
            rv, rz = _topk_ref(oracle_mod, "topk_of", x, k)
            assert np.array_equal(idx.cpu().numpy(), rz)
            assert np.array_equal(vals.cpu().numpy().view(np.int32), rv.view(np.int32))


def _prob_collisions(got_idx, ref_idx, ref_probs_row_fn):
    """Number of rows whose index lists differ; each difference must be a
    probability-rounding collision (values equal within 2 ulp)."""
    diff = 0
    for r in range(got_idx.shape[0]):
        if not np.array_equal(got_idx[r], ref_idx[r]):
            p = ref_probs_row_fn(r)
            a = p[got_idx[r]].astype(np.float64)
            b = p[ref_idx[r]].astype(np.float64)
            assert np.allclose(np.sort(a), np.sort(b), rtol=2.5e-7, atol=0), (r, got_idx[r], ref_idx[r])
            diff += 1
    return diff


@pytest.mark.parametrize("alg,op,base", [
    ("safe_fused", "safe_softmax_fused_topk", "safe_softmax"),
    ("safe_unfused", "safe_softmax_then_topk", "safe_softmax"),
    ("online_unfused", None, "online_softmax"),
])
@pytest.mark.parametrize("shape", ["auto", "split", "warp", "cta"])
def test_probability_selection_topk(cuda, oracle_mod, lib, alg, op, base, shape):
    """Selection on probabilities: indices equal to the reference's except
    where two probabilities collide in fp32 rounding (flagged, counted)."""
    from paper_1805_02867_b200 import osmx

    if shape in ("warp", "cta"):
        lib.config_set("topk_threads", 32 if shape == "warp" else 256)
    else:
        lib.config_set("shape", SHAPES[shape])
    if shape == "split":
        lib.config_set("split_chunk", 2048)
    rng = np.random.default_rng(400)
    collisions = 0
    for V in TOPK_V:
        for d in DISTS:
            k = min(5, V)
            x = dist(d, rng, 5, V)
            vals, idx = osmx.softmax_topk(_dev(x), k, alg=alg)
            y, _ = oracle_mod.batch(base, x)
            if op is None:
                rv, rz = _topk_ref(oracle_mod, "topk_of", y, k)
            else:
                rv, rz = _topk_ref(oracle_mod, op, x, k)
            gi = idx.cpu().numpy()
            if alg == "safe_fused":
                # d in double and the host's expf (csrc/common.cuh expf_ref):
                # keys, hence indices and values, bit for bit (kernels.hpp:95-98)
                assert np.array_equal(gi, rz), (V, d, shape, gi[:2], rz[:2])
                assert np.array_equal(vals.cpu().numpy().view(np.int32), rv.view(np.int32)), (V, d, shape)
            else:  # the unfused pipelines may differ by probability-rounding collisions
                collisions += _prob_collisions(gi, rz, lambda r: y[r])
            assert max_rel(vals.cpu().numpy(), rv) <= TOL
    print(f"{alg}/{shape}: rows with probability-rounding collisions: {collisions}")


def test_topk_known_answers(cuda, lib):
    """SPEC.md:208-233, 294-295 examples and the signed-zero tie probe."""
    from paper_1805_02867_b200 import osmx

    def tk(x, k, alg="online_fused"):
        v, z = osmx.softmax_topk(_dev(np.asarray(x, np.float32).reshape(1, -1)), k, alg=alg)
        return v.cpu().numpy()[0], z.cpu().numpy()[0]

    def to(x, k):
        v, z = osmx.topk(_dev(np.asarray(x, np.float32).reshape(1, -1)), k)
        return v.cpu().numpy()[0], z.cpu().numpy()[0]

    assert list(to([0.1, 0.7, 0.2], 2)[1]) == [1, 2]
    assert list(to([0.5, 0.5], 1)[1]) == [0]
    assert list(to([3, 1, 2], 3)[1]) == [0, 2, 1]
    assert list(to([1, 1, 1], 2)[1]) == [0, 1]
    for alg in ("online_fused", "safe_fused", "safe_unfused", "online_unfused"):
        v, z = tk([1, 2, 3], 2, alg)
        assert list(z) == [2, 1]
        assert abs(v[0] - 0.66524095577482178) <= 1e-6 and abs(v[1] - 0.24472847105479764) <= 1e-6
        v, z = tk([5.0], 1, alg)
        assert list(z) == [0] and v[0] == 1.0
        assert list(tk([2, 2, 1], 2, alg)[1]) == [0, 1]
    assert list(tk([0.0, -0.0, 1.0, 1.0, -0.0, 0.0], 4)[1]) == [2, 3, 0, 1]


def test_nonfinite_rows_flagged(cuda, lib):
    """NaN / +inf / -inf anywhere in a row -> non_finite_error naming the first
    bad row (kernels.hpp:32-35, normalizer.hpp:33)."""
    from paper_1805_02867_b200 import osmx

    rng = np.random.default_rng(5)
    for shape in (0, 1, 2, 3, 4, 5):
        lib.config_set("shape", shape)
        lib.config_set("split_chunk", 2048 if shape == 3 else 0)
        lib.config_set("cluster_size", 2 if shape == 5 else 0)
        for bad in (np.nan, np.inf, -np.inf):
            for V in (7, 3000, 40000):
                if shape in (1, 4) and V > 16384:
                    continue
                x = rng.standard_normal((6, V)).astype(np.float32)
                x[4, V // 2] = bad
                x[5, 0] = bad
                for alg in ("naive", "safe", "online"):
                    with pytest.raises(osmx.NonFiniteError) as e:
                        osmx.softmax(_dev(x), alg=alg)
                    assert e.value.row == 4, (shape, bad, V, alg)
                for alg in ("online_fused", "safe_fused", "safe_unfused", "online_unfused"):
                    with pytest.raises(osmx.NonFiniteError) as e:
                        osmx.softmax_topk(_dev(x), 3, alg=alg)
                    assert e.value.row == 4, (shape, bad, V, alg)
                with pytest.raises(osmx.NonFiniteError):
                    osmx.topk(_dev(x), 3)
        # a clean call afterwards succeeds (the flag was cleared)
        osmx.softmax(_dev(rng.standard_normal((2, 50)).astype(np.float32)))


@pytest.mark.parametrize("shape", ["auto", "resident", "stream", "split", "staged", "cluster"])
def test_nonfinite_at_row_edges(cuda, lib, shape):
    """A single NaN / +inf / -inf at the first or last elements of one row,
    rows at every 16-byte phase (the masked head / tail float4s): that row
    is the one reported."""
    from paper_1805_02867_b200 import osmx

    lib.config_set("shape", SHAPES[shape])
    lib.config_set("split_chunk", 1024 if shape == "split" else 0)
    lib.config_set("cluster_size", 3 if shape == "cluster" else 0)
    rng = np.random.default_rng(17)
    V = 3001
    for phase in range(4):
        big = rng.standard_normal((3, V + 4)).astype(np.float32)
        for pos in (0, 1, 2, V - 2, V - 1):
            for bad in (np.nan, np.inf, -np.inf):
                b = big.copy()
                b[1, phase + pos] = bad
                xt = _dev(b)[:, phase:phase + V]
                for alg in ("naive", "safe", "online"):
                    with pytest.raises(osmx.NonFiniteError) as e:
                        osmx.softmax(xt, alg=alg)
                    assert e.value.row == 1, (shape, phase, pos, bad, alg)
                for alg in ("online_fused", "safe_fused", "safe_unfused", "online_unfused"):
                    with pytest.raises(osmx.NonFiniteError) as e:
                        osmx.softmax_topk(xt, 3, alg=alg)
                    assert e.value.row == 1, (shape, phase, pos, bad, alg)
                with pytest.raises(osmx.NonFiniteError) as e:
                    osmx.topk(xt, 3)
                assert e.value.row == 1, (shape, phase, pos, bad, "topk_of")


def test_argument_errors(cuda, lib):
    from paper_1805_02867_b200 import osmx

    x = _dev(np.zeros((2, 4), np.float32))
    with pytest.raises(osmx.InvalidKError):
        osmx.softmax_topk(x, 0)
    with pytest.raises(osmx.InvalidKError):
        osmx.softmax_topk(x, 5)
    with pytest.raises(osmx.InvalidKError):
        osmx.softmax_topk(_dev(np.zeros((1, 100), np.float32)), 101)
    with pytest.raises(osmx.EmptyInputError):
        osmx.softmax(_dev(np.zeros((2, 0), np.float32)))


@pytest.mark.parametrize("alg", ["online", "safe", "naive"])
def test_softmax_staged_ring_wrap(cuda, oracle_mod, lib, alg):
    """Enough rows per CTA that every slot of the staged ring is refilled
    several times (D = 50 / 12 / 3 slots at V = 1000 / 4099 / 16384), with
    rows of every 16-byte phase."""
    from paper_1805_02867_b200 import osmx

    lib.config_set("shape", SHAPES["staged"])
    rng = np.random.default_rng(11)
    for V, rows in ((1000, 148 * 60), (4099, 148 * 14), (16383, 148 * 5)):
        x = rng.standard_normal((rows, V)).astype(np.float32)
        y = osmx.softmax(_dev(x), alg=alg).cpu().numpy()
        ref, st = oracle_mod.batch(f"{alg}_softmax", x)
        assert (st == 0).all()
        assert max_rel(y, ref) <= TOL, (alg, V)


@pytest.mark.parametrize("variant", ["auto", "warp", "warp_u8", "warp_pf", "warp_pipe1", "warp_pipe3", "warp_db4",
                                     "warp_db2", "warp_bulk"])
def test_online_fused_topk_many_rows(cuda, oracle_mod, lib, variant):
    """Row counts around one wave of warps (the u8 heuristic's range)."""
    from paper_1805_02867_b200 import osmx

    for key, val in TOPK_VARIANTS[variant]:
        lib.config_set(key, val)
    rng = np.random.default_rng(12)
    for rows, V in ((4000, 8192), (2000, 12289)):
        x = dist("quantized2", rng, rows, V) if V == 8192 else dist("normal", rng, rows, V)
        vals, idx = osmx.softmax_topk(_dev(x), 5, alg="online_fused")
        rv, rz = _topk_ref(oracle_mod, "online_softmax_topk", x, 5)
        assert np.array_equal(idx.cpu().numpy(), rz), (variant, rows, V)
        assert max_rel(vals.cpu().numpy(), rv) <= TOL


@pytest.mark.parametrize("variant", ["auto", "split_tma", "split_warp_auto", "split_wide"])
def test_topk_split_more_rows_than_ctas(cuda, oracle_mod, lib, variant):
    """Split records with more rows than resident CTAs (auto: TMA pieces up to
    5 rows per SM, one piece per row, CTAs loop over several rows), misaligned
    rows, fused and topk_of."""
    from paper_1805_02867_b200 import osmx

    for key, val in TOPK_VARIANTS[variant]:
        lib.config_set(key, val)
    rng = np.random.default_rng(13)
    rows, V = 500, 70001
    big = dist("normal", rng, rows, V + 1)
    xt = _dev(big)[:, 1:]  # misaligned rows, ld = V + 1
    x = np.ascontiguousarray(big[:, 1:])
    vals, idx = osmx.softmax_topk(xt, 5, alg="online_fused")
    rv, rz = _topk_ref(oracle_mod, "online_softmax_topk", x, 5)
    assert np.array_equal(idx.cpu().numpy(), rz), variant
    assert max_rel(vals.cpu().numpy(), rv) <= TOL
    tv, ti = osmx.topk(xt, 7)
    qv, qz = _topk_ref(oracle_mod, "topk_of", x, 7)
    assert np.array_equal(ti.cpu().numpy(), qz), variant
    assert np.array_equal(tv.cpu().numpy(), qv)


@pytest.mark.parametrize("alg", ["online", "safe", "naive"])
def test_softmax_cluster_slices(cuda, oracle_mod, lib, alg):
    """Rows split over 2..16 CTAs of a cluster (distributed shared memory
    merge), including empty slices (V < C * 4) and enough rows that every
    ring slot and record parity is reused."""
    from paper_1805_02867_b200 import osmx

    lib.config_set("shape", SHAPES["cluster"])
    rng = np.random.default_rng(13)
    for V, C, rows in ((70001, 0, 300), (16387, 2, 400), (100003, 4, 200), (300001, 16, 48), (5, 4, 33),
                       (40000, 8, 64)):
        lib.config_set("cluster_size", C)
        for d in ("normal", "spikes", "quantized2"):
            x = dist(d, rng, rows, V)
            y = osmx.softmax(_dev(x), alg=alg).cpu().numpy()
            ref, st = oracle_mod.batch(f"{alg}_softmax", x)
            assert (st == 0).all()
            assert max_rel(y, ref) <= TOL, (alg, V, C, d)


@pytest.mark.parametrize("k", [33, 100, 1000, "V"])
def test_large_k(cuda, oracle_mod, lib, k):
    """k above the register lists (radix select + ordered compaction + stable
    segmented sort): indices bit-exact for the raw-key modes, probability
    collisions only for the probability-key modes; k = V sorts whole rows."""
    from paper_1805_02867_b200 import osmx

    rng = np.random.default_rng(500)
    for V in (1000, 4099, 70001):
        kk = V if k == "V" else min(int(k), V)
        if kk == V and V > 5000:
            continue
        for d in ("normal", "quantized2", "equal", "descending", "spikes"):
            x = dist(d, rng, 4, V)
            vals, idx = osmx.softmax_topk(_dev(x), kk, alg="online_fused")
            fv, fz = _topk_ref(oracle_mod, "online_softmax_topk", x, kk)
            assert np.array_equal(idx.cpu().numpy(), fz), (V, kk, d)
            assert max_rel(vals.cpu().numpy(), fv) <= TOL
            tv, ti = osmx.topk(_dev(x), kk)
            rv, rz = _topk_ref(oracle_mod, "topk_of", x, kk)
            assert np.array_equal(ti.cpu().numpy(), rz), (V, kk, d)
            assert np.array_equal(tv.cpu().numpy().view(np.int32), rv.view(np.int32))
            if V == 4099 and d == "normal":  # the reference-shaped host API (numpy in/out), same device path
                r = osmx.online_softmax_topk(x, kk)
                assert np.array_equal(np.asarray(r.indices), fz)
                assert max_rel(np.asarray(r.values), fv) <= TOL
            for alg, op in (("safe_fused", "safe_softmax_fused_topk"), ("safe_unfused", "safe_softmax_then_topk")):
                vals, idx = osmx.softmax_topk(_dev(x), kk, alg=alg)
                y, _ = oracle_mod.batch("safe_softmax", x)
                rv, rz = _topk_ref(oracle_mod, op, x, kk)
                _prob_collisions(idx.cpu().numpy(), rz, lambda r: y[r])
                assert max_rel(vals.cpu().numpy(), rv) <= TOL


def _collision_rows(rng, rows, V):
    """Rows whose top probabilities collide after float rounding: 64 distinct
    logits 1 - j*2^-24 (j < 64) at random positions over a normal background.
    Their e^(x - m) are distinct floats just below 1, but divided by d they
    round onto a coarser grid, so several share one p and the reference's
    tie rule (lowest index first, topk.hpp:37-43) decides the order."""
    # background capped below the 64 planted logits, so they are the top
    x = np.minimum(rng.standard_normal((rows, V)) * 2.0 - 6.0, -1.0).astype(np.float32)
    for r in range(rows):
        pos = rng.choice(V, size=min(64, V), replace=False)
        x[r, pos] = (1.0 - np.arange(len(pos)) * 2.0 ** -24).astype(np.float32)
    return x


@pytest.mark.parametrize("shape", ["auto", "split", "warp", "cta"])
@pytest.mark.parametrize("V", [100, 5003, 70001, 300000])
def test_safe_fused_topk_collisions_bit_exact(cuda, oracle_mod, lib, shape, V):
    """safe_softmax_fused_topk selects on float(expf(x - m) / d) with a double
    d (kernels.hpp:95-98): with colliding probabilities only the reference's
    exact arithmetic reproduces its indices.  k = 5, 32 and (large-k path) 40."""
    from paper_1805_02867_b200 import osmx

    if shape in ("warp", "cta"):
        lib.config_set("topk_threads", 32 if shape == "warp" else 256)
    else:
        lib.config_set("shape", SHAPES[shape])
    rng = np.random.default_rng(V)
    x = _collision_rows(rng, 4, V)
    for k in (5, 32, 40):
        if k > V:
            continue
        vals, idx = osmx.softmax_topk(_dev(x), k, alg="safe_fused")
        rv, rz = _topk_ref(oracle_mod, "safe_softmax_fused_topk", x, k)
        assert np.array_equal(idx.cpu().numpy(), rz), (k, shape)
        assert np.array_equal(vals.cpu().numpy().view(np.int32), rv.view(np.int32)), (k, shape)
        # the collisions are real: some selected probabilities are equal (at
        # V = 100 the planted values' quotients land on distinct floats)
        if V >= 5003:
            assert (np.diff(rv, axis=1) == 0).any()


@pytest.mark.parametrize("k", [33, 257, 4096])
def test_large_k_fast_path_edges(cuda, oracle_mod, lib, k):
    """The two-pass large-k path (csrc/topk_large.cu k_topk_large_fast):
    a boundary bucket too full for shared memory (every key with the same
    top 11 bits: the radix fallback), signed zeros kept in topk_of values,
    candidates arriving in any order (bucket ties broken by index)."""
    from paper_1805_02867_b200 import osmx

    rng = np.random.default_rng(900 + k)
    V = 20011
    narrow = (1.0 + rng.random((3, V)) * 1e-3).astype(np.float32)  # one top-11-bit bucket
    zeros = np.zeros((3, V), dtype=np.float32)
    zeros[:, rng.choice(V, size=V // 2, replace=False)] = -0.0
    spiky = rng.standard_normal((3, V)).astype(np.float32)
    spiky[:, ::7] = 3.0  # many equal keys inside the boundary bucket
    for x in (narrow, zeros, spiky):
        vals, idx = osmx.softmax_topk(_dev(x), k, alg="online_fused")
        fv, fz = _topk_ref(oracle_mod, "online_softmax_topk", x, k)
        assert np.array_equal(idx.cpu().numpy(), fz)
        assert max_rel(vals.cpu().numpy(), fv) <= TOL
        tv, ti = osmx.topk(_dev(x), k)
        rv, rz = _topk_ref(oracle_mod, "topk_of", x, k)
        assert np.array_equal(ti.cpu().numpy(), rz)
        assert np.array_equal(tv.cpu().numpy().view(np.int32), rv.view(np.int32))
