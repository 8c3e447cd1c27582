"""Generate tests/golden/golden.npz from the REFERENCE implementation itself.

Run in the authoring container (needs oracle/_ref/libosmx_ref.so, built by
oracle/Makefile from /root/reference/proj/src with -Dosmx=osmx_ref):

    python tests/golden/make_golden.py

Every case is a seeded input row; the outputs are what the unmodified
reference returns for it (naive/safe/online softmax, the four top-K entry
points and topk_of, oracle_softmax, run_normalizer<float/double> and the
chunked normalizer).  The fixtures travel with the repo, so the CPU and GPU
parity tests never need /root/reference at run time.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402
from tests._util import dist  # noqa: E402

CASES = [
    # (name, distribution, V, k, seed)
    ("v1", "normal", 1, 1, 1),
    ("v2_tie", "equal", 2, 1, 2),
    ("v3", "normal", 3, 2, 3),
    ("v5_q", "quantized2", 5, 5, 4),
    ("v17_spikes", "spikes", 17, 5, 5),
    ("v64_asc", "ascending", 64, 5, 6),
    ("v64_desc", "descending", 64, 5, 7),
    ("v100_q100", "quantized100", 100, 5, 8),
    ("v257_wide", "wide", 257, 8, 9),
    ("v1000_normal", "normal", 1000, 5, 10),
    ("v1023_q2", "quantized2", 1023, 13, 11),
    ("v2049_normal", "normal", 2049, 32, 12),
    ("v4099_q100", "quantized100", 4099, 5, 13),
]

SOFTMAX = ["naive_softmax", "safe_softmax", "online_softmax"]
TOPK = ["safe_softmax_then_topk", "safe_softmax_fused_topk", "online_softmax_topk", "topk_of", "oracle_topk"]


def main() -> None:
    assert O.ref_available(), "build oracle/_ref first (make -C oracle)"
    out = {}
    for name, d, V, k, seed in CASES:
        rng = np.random.default_rng(seed)
        x = dist(d, rng, 1, V)[0]
        out[f"{name}/x"] = x
        out[f"{name}/k"] = np.int64(k)
        for op in SOFTMAX:
            y, st = O.softmax(op, x, impl="ref")
            assert st == 0
            out[f"{name}/{op}"] = y
        for op in TOPK:
            v, z, st = O.topk(op, x, k, impl="ref")
            assert st == 0
            out[f"{name}/{op}/values"] = v
            out[f"{name}/{op}/indices"] = z
        ys, st = O.softmax_double(x, impl="ref")
        out[f"{name}/oracle_softmax"] = ys
        for dbl in (0, 1):
            m, dd, st = O.normalizer(x, dbl=bool(dbl), impl="ref")
            out[f"{name}/run_normalizer_{'double' if dbl else 'float'}"] = np.array([m, dd])
            m, dd, st = O.normalizer(x, dbl=bool(dbl), chunk=7, impl="ref")
            out[f"{name}/run_normalizer_chunked7_{'double' if dbl else 'float'}"] = np.array([m, dd])
    # the reference's own generator (bench.cpp:162-172), seed 1, batch 3 x 10
    out["generate_inputs/seed1_3x10"] = O.generate_inputs(1, 3, 10)
    out["log_spaced_sizes/10_1e6_21"] = np.array(O.log_spaced_sizes(10, 1000000, 21))
    counts = []
    for alg in range(6):
        for v in (100, 1000, 100000):
            k = 5 if alg >= 3 else 0
            lo, stt, s = O.count_accesses(alg, v, k, impl="ref")
            counts.append((alg, v, k, lo, stt))
    out["count_accesses"] = np.array(counts, dtype=np.int64)
    np.savez_compressed(Path(__file__).with_name("golden.npz"), **out)
    print(f"wrote {len(out)} arrays")


if __name__ == "__main__":
    main()
