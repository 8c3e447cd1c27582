"""bench.py's JSON line contract (driver-facing keys), both arms."""
from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def _run(args, timeout=900):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    # the driver keeps only the tail of stdout: the headline must be the
    # LAST line and short enough to survive in full
    assert lines and len(lines[-1].encode()) < 2048, out.stdout[-3000:]
    return json.loads(lines[-1])


def test_reference_arm_line():
    """--impl reference: the reference CPU library on the host cores."""
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--rows", "16", "--V", "4096"])
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


@pytest.mark.gpu
def test_our_arm_line():
    d = _run(["--rows", "512", "--V", "16384", "--steps", "3", "--warmup", "3", "--sweep", "off", "--cpu", "off"])
    assert BASE_KEYS <= set(d)
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["gpu_launches"] == 3
    assert d["e2e"]["steps"] == 3  # e2e honours --steps
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["peak"] > 0 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    assert d["e2e"]["h2d_bytes_per_step"] == 512 * 16384 * 4 and d["e2e"]["consistent"] is True
    assert d["parity"]["idx_exact"] is True and d["parity"]["max_rel_err"] <= 1e-5
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    assert r["read_probe_GBps"] > 0 and 0 < r["frac_of_read_probe"] < 1.5


def test_compact_line_bounded():
    """The headline line stays < 2 KB even with every optional block filled."""
    sys.path.insert(0, str(ROOT))
    import bench

    big = {k: "x" * 20 for k in BASE_KEYS}
    big.update({"value": 1.0, "config": {"workload": "w" * 200}, "clocks": {"sm_mhz": 1, "sm_max_mhz": 2,
                                                                          "reasons": ["a"], "samples": 3},
                "roofline": {"bound": "hbm", "achieved": 1, "peak": 2, "unit": "GB/s", "frac": 0.5, "traffic": 3,
                             "kernel": "k" * 3000},
                "e2e": {"value": 1, "unit": "GB/s", "h2d_bytes_per_step": 1, "d2h_bytes_per_step": 1,
                        "notes": "n" * 3000},
                "cpu_baseline": {"value": 1, "unit": "GB/s", "cores": 1, "kind": "reference", "sample": "s" * 300},
                "parity": {"rows_checked": 8, "indices_bit_exact": True, "max_rel_err": 1e-7},
                "sweep": {"softmax": [], "topk": [], "c5": {"online_fused": {"ms": 1, "frac": 1}}}})
    line = bench.compact_line(big)
    s = json.dumps(line, separators=(",", ":"))
    assert len(s) <= bench.FINAL_LINE_MAX
    assert {"roofline", "e2e", "cpu_baseline", "clocks"} <= set(line)
