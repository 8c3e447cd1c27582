"""Kernel-shape tuning sweep (cold L2 between repeats): for each V, time every
kernel family the launch layer could pick, so the heuristics in
csrc/softmax_impl.cuh / topk_impl.cuh are set from measurements.

    python tools/shape_sweep.py --rows 4000 --alg online --V 1000 3162 10000
    python tools/shape_sweep.py --rows 4000 --alg online_fused --V 32768 --knob topk_threads=32,128
"""
from __future__ import annotations

import argparse
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from bench import algo_bytes, n_rotating_sets, time_rotating  # noqa: E402
from paper_1805_02867_b200 import _lib  # noqa: E402

DEFAULTS = {"resident_max_v": 2048, "tma": 0, "topk_u8": -1, "l2_prefetch": -1, "topk_pipe": 0, "split_cta": -1, "staged_kb": 0, "staged_gw": 0, "staged_ng": 0, "stream_ctas": 0, "cluster_size": 0, "stream_threads": 0}
IDS = {"naive": 0, "safe": 1, "online": 2, "safe_unfused": 3, "safe_fused": 4, "online_fused": 5,
       "online_unfused": 6}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=4000)
    ap.add_argument("--alg", nargs="+", default=["online"])
    ap.add_argument("--V", type=int, nargs="+", default=[1000, 3162, 10000])
    ap.add_argument("--k", type=int, default=5)
    ap.add_argument("--reps", type=int, default=9)
    ap.add_argument("--knob", action="append", default=[], help="key=v1,v2,...")
    ap.add_argument("--set", action="append", default=[], help="key=v fixed for the whole run")
    a = ap.parse_args()
    lib = _lib.load()
    for kv in a.set:
        _lib.config_set(kv.split("=")[0], int(kv.split("=")[1]))
    dev = torch.device("cuda", 0)
    sp = torch.cuda.current_stream().cuda_stream
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    knobs = [(kv.split("=")[0], [int(v) for v in kv.split("=")[1].split(",")]) for kv in a.knob] or [("shape", [0])]
    out = []
    for V in a.V:
        nset = n_rotating_sets(8 * a.rows * V, l2, cap_bytes=24 << 30)
        x = torch.empty((nset, a.rows, V), device=dev).normal_()
        y = torch.empty_like(x) if any(IDS[n] < 3 for n in a.alg) else None
        vals = torch.empty((a.rows, a.k), device=dev)
        idx = torch.empty((a.rows, a.k), dtype=torch.int64, device=dev)
        for alg_name in a.alg:
            alg = IDS[alg_name]
            topk = alg >= 3
            for key, values in knobs:
                for val in values:
                    _lib.config_set(key, val)
                    nb = lib.osmx_workspace_bytes(alg, a.rows, V, a.k if topk else 0)
                    ws = torch.zeros(max(nb, 256), dtype=torch.uint8, device=dev)

                    def launch(i, st):
                        if topk:
                            r = lib.osmx_softmax_topk(alg, x[i].data_ptr(), V, a.rows, V, a.k, vals.data_ptr(),
                                                      idx.data_ptr(), ws.data_ptr(), ws.numel(), st)
                        else:
                            r = lib.osmx_softmax(alg, x[i].data_ptr(), V, y[i].data_ptr(), V, a.rows, V,
                                                 ws.data_ptr(), ws.numel(), st)
                        if r != 0:
                            raise RuntimeError(f"status {r}")

                    try:
                        launch(0, sp)
                        torch.cuda.synchronize()
                    except RuntimeError as e:  # layout not launchable for this V
                        print(json.dumps({"V": V, "alg": alg_name, key: val, "error": str(e)}), flush=True)
                        _lib.config_set(key, DEFAULTS.get(key, 0))
                        continue
                    ms, ms_min = time_rotating(launch, nset, a.reps)
                    gbs = algo_bytes(alg_name, a.rows, V, a.k) / (ms * 1e-3) / 1e9
                    dram = (8 * a.rows * V if not topk else 4 * a.rows * V) / (ms * 1e-3) / 1e9
                    rec = {"V": V, "alg": alg_name, key: val, "ms": round(ms, 4), "GBps": round(gbs, 1),
                           "dram_floor_GBps": round(dram, 1)}
                    out.append(rec)
                    print(json.dumps(rec), flush=True)
                    del ws
                _lib.config_set(key, DEFAULTS.get(key, 0))
        del x, y
    return out


if __name__ == "__main__":
    main()
