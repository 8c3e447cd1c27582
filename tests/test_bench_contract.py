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
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


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
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["peak"] > 0 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    assert d["e2e"]["h2d_bytes_per_step"] == 512 * 16384 * 4 and d["e2e"]["consistent"] is True
    assert d["parity"]["indices_bit_exact"] is True and d["parity"]["max_rel_err"] <= 1e-5
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    assert r["read_probe_GBps"] > 0 and 0 < r["frac_of_read_probe"] < 1.5
