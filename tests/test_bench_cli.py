"""osmx-bench-gpu (tools/osmx_bench_gpu.cu): the reference CLI's flags and
table (tools/osmx_bench.cpp:65-84, bench.cpp:223-253) on the B200 kernels.
The counts-only table needs no GPU and is checked against the oracle's
access model (itself pinned to the reference, test_oracle.py)."""
from __future__ import annotations

import io
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
CLI = ROOT / "build" / "osmx-bench-gpu"
COLS = ["NaiveSoftmax", "SafeSoftmax", "OnlineSoftmax", "SafeSoftmaxUnfusedTopK", "SafeSoftmaxFusedTopK",
        "OnlineSoftmaxFusedTopK"]


@pytest.fixture(scope="module")
def cli():
    if not CLI.exists():
        subprocess.run(["make", "-C", str(ROOT), "benchcli"], check=True, capture_output=True)
    return CLI


def parse(text: str, delim: str = ","):
    lines = [ln for ln in text.splitlines() if ln and not ln.startswith("#")]
    header = lines[0].split(delim)
    rows = [[float(c) for c in ln.split(delim)] for ln in lines[1:]]
    return header, np.array(rows)


def test_counts_only_matches_access_model(cli, oracle_mod):
    out = subprocess.run([str(cli), "--counts-only", "--vmin", "10", "--vmax", "1000000", "--points", "21",
                          "--k", "5"], capture_output=True, text=True, check=True).stdout
    header, rows = parse(out)
    assert header[0] == "V"
    assert header[1:] == [f"{c}_{s}" for c in COLS for s in ("loads", "stores")]  # no throughput / ratios
    assert [int(v) for v in rows[:, 0]] == list(oracle_mod.log_spaced_sizes(10, 1000000, 21))
    for r in rows:
        V = int(r[0])
        for a, col in enumerate(COLS):
            lo, st, _ = oracle_mod.count_accesses(a, V, 5 if a >= 3 else 0)
            i = header.index(f"{col}_loads")
            assert (r[i], r[i + 1]) == (lo, st), (V, col)


def test_flags_and_errors(cli):
    out = subprocess.run([str(cli), "--counts-only", "--sizes", "7,3,7", "--algorithms", "online,SafeSoftmax",
                          "--format", "tsv"], capture_output=True, text=True, check=True).stdout
    header, rows = parse(out, "\t")
    assert header == ["V", "OnlineSoftmax_loads", "OnlineSoftmax_stores", "SafeSoftmax_loads", "SafeSoftmax_stores"]
    assert list(rows[:, 0]) == [3, 7]  # sorted, deduplicated (bench.cpp run_sweep)
    bad = subprocess.run([str(cli), "--algorithms", "fastest"], capture_output=True, text=True)
    assert bad.returncode == 2 and "unknown algorithm" in bad.stderr
    both = subprocess.run([str(cli), "--sizes", "10", "--vmin", "5"], capture_output=True, text=True)
    assert both.returncode == 2


@pytest.mark.gpu
def test_timed_sweep_on_device(cli, tmp_path):
    p = tmp_path / "sweep.csv"
    subprocess.run([str(cli), "--sizes", "1000,4099", "--batch", "64", "--repeats", "3", "--out", str(p),
                    "--plot", str(tmp_path / "plt"), "--algorithms",
                    "naive,safe,online,safe-unfused-topk,safe-fused-topk,online-fused-topk,online-unfused-topk"],
                   check=True, capture_output=True, text=True)
    header, rows = parse(p.read_text())
    for col in COLS + ["OnlineSoftmaxUnfusedTopK", "OnlineSoftmax_over_SafeSoftmax",
                       "OnlineSoftmaxFusedTopK_over_SafeSoftmaxUnfusedTopK", "OnlineSoftmaxFusedTopK_GBps"]:
        assert col in header, col
        assert np.isfinite(rows[:, header.index(col)]).all() and (rows[:, header.index(col)] > 0).all()
    assert (tmp_path / "plt.OnlineSoftmax.dat").exists()
