"""Measured DRAM bytes for every cell of bench.py's sweeps.

    # on the GPU box: run the cells once under ncu (one pass, caches as left
    # by the previous step -- L2 is flushed by a 512 MB write before each cell,
    # like the sweep's rotating cold buffers)
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --cache-control none --clock-control none --csv --log-file gpurun_out/cells.csv \
        python tools/dram_cells.py run --out gpurun_out/cells_plan.json
    # anywhere: attribute the launches to the cells -> profiles/dram_cells_rNN.json
    python tools/dram_cells.py merge gpurun_out/cells_plan.json gpurun_out/cells.csv profiles/dram_cells_r02.json
    # optional: append <alg>_dram_bytes columns to an osmx-bench-gpu CSV
    python tools/dram_cells.py csv profiles/dram_cells_r02.json build_out.csv > with_dram.csv

The plan file lists, in launch order, each cell's (alg, V, rows) and how many
of this library's kernels it launched (osmx_launch_count before / after);
`merge` walks the ncu launch list (this library's kernels only: the
anonymous-namespace k_* names) in the same order and sums each cell's DRAM
read + write bytes.  bench.py reads the result and prints `dram_bytes` and a
DRAM-based `dram_frac` next to every cell's algorithmic `frac`.
"""
from __future__ import annotations

import argparse
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

B = 4000
K = 5
SOFTMAX = (("naive", 0, 0), ("safe", 1, 0), ("online", 2, 0), ("safe_stream", 1, 2), ("online_stream", 2, 2))
TOPK = (("online_fused", 5, 0), ("online_unfused", 6, 0), ("safe_unfused", 3, 0), ("safe_fused", 4, 0),
        ("online_unfused_stream", 6, 2))


def run(out: str) -> None:
    import torch

    from bench import Vs_all, Vt_all
    from paper_1805_02867_b200 import _lib

    lib = _lib.load()
    dev = torch.device("cuda", 0)
    sp = torch.cuda.current_stream().cuda_stream
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    plan = []

    def cell(name, V, rows, fn):
        flush.zero_()  # evict the inputs' tail that generation left in L2
        torch.cuda.synchronize()
        n0 = lib.osmx_launch_count()
        assert fn() == 0, name
        torch.cuda.synchronize()
        plan.append({"alg": name, "V": V, "rows": rows, "launches": int(lib.osmx_launch_count() - n0)})

    for V in Vs_all:
        x = torch.empty((B, V), device=dev).normal_()
        y = torch.empty_like(x)
        for name, alg, shape in SOFTMAX:
            _lib.config_set("shape", shape)
            ws = torch.zeros(lib.osmx_workspace_bytes(alg, B, V, 0), dtype=torch.uint8, device=dev)
            cell(name, V, B, lambda: lib.osmx_softmax(alg, x.data_ptr(), V, y.data_ptr(), V, B, V, ws.data_ptr(),
                                                      ws.numel(), sp))
            _lib.config_set("shape", 0)
        del x, y
    vals = torch.empty((B, K), device=dev)
    idx = torch.empty((B, K), dtype=torch.int64, device=dev)
    for V in sorted(set(Vs_all) | set(Vt_all)):  # the CLI's grid and configs[2]
        x = torch.empty((B, V), device=dev).normal_()
        for name, alg, shape in TOPK:
            _lib.config_set("shape", shape)
            ws = torch.zeros(lib.osmx_workspace_bytes(alg, B, V, K), dtype=torch.uint8, device=dev)
            cell(name, V, B, lambda: lib.osmx_softmax_topk(alg, x.data_ptr(), V, B, V, K, vals.data_ptr(),
                                                           idx.data_ptr(), ws.data_ptr(), ws.numel(), sp))
            _lib.config_set("shape", 0)
        del x
    # configs[4]: one row of 2^26
    V = 1 << 26
    x = torch.empty((1, V), device=dev).normal_()
    y = torch.empty_like(x)
    ws = torch.zeros(max(lib.osmx_workspace_bytes(5, 1, V, K), lib.osmx_workspace_bytes(2, 1, V, 0)),
                     dtype=torch.uint8, device=dev)
    cell("c5_online_fused", V, 1, lambda: lib.osmx_softmax_topk(5, x.data_ptr(), V, 1, V, K, vals.data_ptr(),
                                                                idx.data_ptr(), ws.data_ptr(), ws.numel(), sp))
    cell("c5_online", V, 1, lambda: lib.osmx_softmax(2, x.data_ptr(), V, y.data_ptr(), V, 1, V, ws.data_ptr(),
                                                     ws.numel(), sp))
    Path(out).write_text(json.dumps({"batch": B, "k": K, "cells": plan}, indent=1))
    print(f"{len(plan)} cells, {sum(c['launches'] for c in plan)} launches")


def ncu_launches(path: str):
    """[(kernel name, {metric: value})] in launch order, this library's kernels only."""
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hdr]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    ui = h.index("Metric Unit")
    out = {}
    for r in rows[hdr + 1:]:
        if len(r) != len(h) or "<unnamed>::k_" not in r[ki]:
            continue
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9,
                 "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1.0, "s": 1.0}[r[ui]]
        out.setdefault(int(r[ii]), [r[ki], {}])[1][r[mi]] = float(r[vi].replace(",", "")) * scale
    return [out[i] for i in sorted(out)]


def merge(plan_path: str, csv_path: str, out: str) -> None:
    plan = json.loads(Path(plan_path).read_text())
    launches = ncu_launches(csv_path)
    need = sum(c["launches"] for c in plan["cells"])
    if need != len(launches):
        raise SystemExit(f"plan has {need} launches, the ncu list {len(launches)}")
    from bench import algo_bytes

    i = 0
    cells = []
    for c in plan["cells"]:
        ks = launches[i:i + c["launches"]]
        i += c["launches"]
        rd = sum(m.get("dram__bytes_read.sum", 0.0) for _, m in ks)
        wr = sum(m.get("dram__bytes_write.sum", 0.0) for _, m in ks)
        t = sum(m.get("gpu__time_duration.sum", 0.0) for _, m in ks)
        base = c["alg"].replace("c5_", "").replace("_stream", "")
        algo = algo_bytes(base, c["rows"], c["V"], plan["k"])
        cells.append({**c, "dram_read": int(rd), "dram_write": int(wr), "dram_bytes": int(rd + wr),
                      "algo_bytes": int(algo), "dram_over_algo": round((rd + wr) / algo, 4),
                      "ncu_kernel_ms": round(t * 1e3, 5), "kernels": [n.split("(")[0] for n, _ in ks]})
    Path(out).write_text(json.dumps({"source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,"
                                               "gpu__time_duration.sum --cache-control none (L2 flushed by a "
                                               "512 MB write before each cell), tools/dram_cells.py",
                                     "batch": plan["batch"], "k": plan["k"], "cells": cells}, indent=1))
    print(f"{len(cells)} cells -> {out}")


CLI_NAMES = {"naive": "NaiveSoftmax", "safe": "SafeSoftmax", "online": "OnlineSoftmax",
             "safe_unfused": "SafeSoftmaxUnfusedTopK", "safe_fused": "SafeSoftmaxFusedTopK",
             "online_fused": "OnlineSoftmaxFusedTopK", "online_unfused": "OnlineSoftmaxUnfusedTopK"}


def to_csv(cells_path: str, bench_csv: str) -> None:
    """Append <Algorithm>_dram_bytes columns (measured DRAM bytes per vector,
    the ncu counterpart of the access-model _loads/_stores columns) to an
    osmx-bench-gpu CSV; comment lines pass through."""
    cells = json.loads(Path(cells_path).read_text())["cells"]
    by = {(CLI_NAMES[c["alg"]], c["V"]): c["dram_bytes"] / c["rows"] for c in cells if c["alg"] in CLI_NAMES}
    algs = [CLI_NAMES[a] for a in CLI_NAMES]
    w = csv.writer(sys.stdout, lineterminator="\n")
    header = None
    for r in csv.reader(open(bench_csv)):
        if not r or r[0].startswith("#"):
            sys.stdout.write(",".join(r) + "\n")
            continue
        if header is None:
            header = r
            w.writerow(r + [f"{a}_dram_bytes" for a in algs])
            continue
        V = int(float(r[0]))
        w.writerow(r + [("%.1f" % by[(a, V)]) if (a, V) in by else "" for a in algs])


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("run")
    p.add_argument("--out", required=True)
    p = sub.add_parser("merge")
    p.add_argument("plan")
    p.add_argument("ncu_csv")
    p.add_argument("out")
    p = sub.add_parser("csv")
    p.add_argument("cells")
    p.add_argument("bench_csv")
    a = ap.parse_args()
    if a.cmd == "run":
        run(a.out)
    elif a.cmd == "merge":
        merge(a.plan, a.ncu_csv, a.out)
    else:
        to_csv(a.cells, a.bench_csv)
