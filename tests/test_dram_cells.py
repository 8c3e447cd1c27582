"""tools/dram_cells.py: ncu launch attribution to sweep cells and the
measured-DRAM columns bench.py / the CLI CSV carry (CPU only)."""
from __future__ import annotations

import csv
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def _ncu_csv(path: Path, launches):
    """A --csv --metrics launch list in ncu's layout: one row per metric."""
    hdr = ["ID", "Process ID", "Process Name", "Host Name", "Kernel Name", "Context", "Stream", "Block Size",
           "Grid Size", "Device", "CC", "Section Name", "Metric Name", "Metric Unit", "Metric Value"]
    with open(path, "w", newline="") as f:
        f.write("==PROF== Connected to process 1\n")
        w = csv.writer(f, quoting=csv.QUOTE_ALL)
        w.writerow(hdr)
        for i, (name, rd, wr, ns) in enumerate(launches):
            for m, u, v in (("dram__bytes_read.sum", "Mbyte", rd / 1e6), ("dram__bytes_write.sum", "Mbyte", wr / 1e6),
                            ("gpu__time_duration.sum", "nsecond", ns)):
                w.writerow([i, 1, "python", "h", name, 1, 7, "(1,1,1)", "(1,1,1)", 0, "10.0",
                            "Command line profiler metrics", m, u, f"{v:,.3f}" if u != "nsecond" else str(v)])


def test_merge_attributes_launches_in_order(tmp_path):
    plan = {"batch": 4000, "k": 5, "cells": [
        {"alg": "online", "V": 1000, "rows": 4000, "launches": 1},
        {"alg": "online_unfused", "V": 1000, "rows": 4000, "launches": 2},
        {"alg": "online_fused", "V": 1000, "rows": 4000, "launches": 1}]}
    (tmp_path / "plan.json").write_text(json.dumps(plan))
    ours = "void <unnamed>::k_softmax_staged<1>(const float *)"
    _ncu_csv(tmp_path / "l.csv", [
        ("void at::native::normal_kernel(float*)", 9e9, 9e9, 1),  # torch: skipped
        (ours, 16e6, 16e6, 1000), (ours, 16e6, 16e6, 1000),
        ("void <unnamed>::k_topk_rows<32>(const float *)", 16e6, 0.1e6, 900),
        ("void <unnamed>::k_topk_rows<32>(const float *)", 16e6, 0.2e6, 800)])
    out = tmp_path / "cells.json"
    subprocess.run([sys.executable, str(ROOT / "tools/dram_cells.py"), "merge", str(tmp_path / "plan.json"),
                    str(tmp_path / "l.csv"), str(out)], check=True, cwd=ROOT)
    cells = json.loads(out.read_text())["cells"]
    assert [c["dram_bytes"] for c in cells] == [32_000_000, 48_100_000, 16_200_000]
    assert cells[0]["algo_bytes"] == 4000 * 12 * 1000
    assert abs(cells[1]["ncu_kernel_ms"] - 1.9e-3) < 1e-9

    # the CLI CSV gets <Algorithm>_dram_bytes (per vector) columns
    cli = tmp_path / "cli.csv"
    cli.write_text("# generated: x\nV,OnlineSoftmax,OnlineSoftmaxFusedTopK\n1000,1.0,2.0\n10,3.0,4.0\n")
    r = subprocess.run([sys.executable, str(ROOT / "tools/dram_cells.py"), "csv", str(out), str(cli)],
                       check=True, capture_output=True, text=True, cwd=ROOT)
    lines = r.stdout.splitlines()
    assert lines[0].startswith("# generated")
    head = lines[1].split(",")
    row = dict(zip(head, lines[2].split(",")))
    assert row["OnlineSoftmax_dram_bytes"] == "8000.0" and row["OnlineSoftmaxFusedTopK_dram_bytes"] == "4050.0"
    assert dict(zip(head, lines[3].split(",")))["OnlineSoftmax_dram_bytes"] == ""


def test_bench_reads_measured_cells(tmp_path, monkeypatch):
    sys.path.insert(0, str(ROOT))
    import bench

    prof = tmp_path / "profiles"
    prof.mkdir()
    (prof / "dram_cells_r02.json").write_text(json.dumps({"cells": [
        {"alg": "online", "V": 1000, "dram_bytes": 32_000_000}]}))
    monkeypatch.setattr(bench, "ROOT", tmp_path)
    d = bench.dram_cells()
    assert d[("online", 1000)] == 32_000_000 and d["_source"] == "dram_cells_r02.json"
    cell = {"ms": 0.01}
    bench.add_dram(cell, d, "online", 1000, 0.01, 6400.0)
    assert cell["dram_bytes"] == 32_000_000 and cell["dram_frac"] == 0.5
