"""Run one C-ABI op a few times (for ncu captures and quick timing).

    python tools/run_op.py --alg online_fused --rows 4096 --V 131072 --k 5 --reps 3 [--set tma=2 ...]

Prints the CUDA-event time per launch (median) and algorithmic GB/s.
"""
from __future__ import annotations

import argparse
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from bench import algo_bytes, measured_peaks  # noqa: E402
from paper_1805_02867_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--alg", default="online_fused")
    ap.add_argument("--rows", type=int, default=4096)
    ap.add_argument("--V", type=int, default=131072)
    ap.add_argument("--k", type=int, default=5)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--set", action="append", default=[])
    a = ap.parse_args()
    lib = _lib.load()
    for kv in a.set:
        key, val = kv.split("=")
        _lib.config_set(key, int(val))
    ids = {"naive": 0, "safe": 1, "online": 2, "safe_unfused": 3, "safe_fused": 4, "online_fused": 5,
           "online_unfused": 6}
    alg = ids[a.alg]
    dev = torch.device("cuda", 0)
    x = torch.empty((a.rows, a.V), device=dev).normal_()
    sp = torch.cuda.current_stream().cuda_stream
    topk = alg >= 3
    nb = lib.osmx_workspace_bytes(alg, a.rows, a.V, a.k if topk else 0)
    ws = torch.zeros(max(nb, 256), dtype=torch.uint8, device=dev)
    if topk:
        vals = torch.empty((a.rows, a.k), device=dev)
        idx = torch.empty((a.rows, a.k), dtype=torch.int64, device=dev)

        def fn():
            return lib.osmx_softmax_topk(alg, x.data_ptr(), a.V, a.rows, a.V, a.k, vals.data_ptr(), idx.data_ptr(),
                                         ws.data_ptr(), ws.numel(), sp)
    else:
        y = torch.empty_like(x)

        def fn():
            return lib.osmx_softmax(alg, x.data_ptr(), a.V, y.data_ptr(), a.V, a.rows, a.V, ws.data_ptr(),
                                    ws.numel(), sp)
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st = fn()
        e1.record()
        e1.synchronize()
        assert st == 0, _lib.status_string(st)
        ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    gbs = algo_bytes(a.alg, a.rows, a.V, a.k) / (ms * 1e-3) / 1e9
    print(f"{a.alg} rows={a.rows} V={a.V} k={a.k} {a.set}: {ms:.4f} ms  {gbs:.1f} GB/s  "
          f"frac={gbs / measured_peaks()['hbm_gbs']:.3f}")


if __name__ == "__main__":
    main()
