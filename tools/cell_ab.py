"""Same-box A/B of launch knobs on one sweep cell, timed like bench.py's sweeps
(rotating cold buffer sets, one CUDA graph, CUDA events, median), settings
interleaved over several rounds so clock drift hits every setting alike.

    python tools/cell_ab.py --alg online_fused --rows 4000 --V 32768 \
        --cfg topk_block=32 --cfg topk_block=128 [--rounds 3]
A --cfg takes comma-separated key=value knobs ("" = library defaults)."""
from __future__ import annotations

import argparse
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from bench import Arena, algo_bytes, measured_peaks, n_rotating_sets, time_rotating  # noqa: E402
from paper_1805_02867_b200 import _lib  # noqa: E402

IDS = {"naive": 0, "safe": 1, "online": 2, "safe_unfused": 3, "safe_fused": 4, "online_fused": 5, "online_unfused": 6}


def main():
    import faulthandler
    import os

    if os.environ.get("OSMX_WATCHDOG"):  # dump every thread's stack if a run hangs
        faulthandler.dump_traceback_later(int(os.environ["OSMX_WATCHDOG"]), exit=True)
    ap = argparse.ArgumentParser()
    ap.add_argument("--alg", default="online_fused")
    ap.add_argument("--rows", type=int, default=4000)
    ap.add_argument("--V", type=int, default=32768)
    ap.add_argument("--k", type=int, default=5)
    ap.add_argument("--cfg", action="append", default=[])
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    lib = _lib.load()
    dev = torch.device("cuda", 0)
    alg, B, V, k = IDS[a.alg], a.rows, a.V, a.k
    topk = alg >= 3
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    n = n_rotating_sets((4 if topk else 8) * B * V, l2)
    arena = Arena(2 * n * B * V, dev)
    x = arena.take(0, (n, B, V)).normal_()
    y = arena.take(n * B * V, (n, B, V))
    vals = torch.empty((B, k), device=dev)
    idx = torch.empty((B, k), dtype=torch.int64, device=dev)
    cfgs = a.cfg or [""]
    res = {c: [] for c in cfgs}
    peak = measured_peaks()["hbm_gbs"]
    for _ in range(a.rounds):
        for c in cfgs:
            kv = [p.split("=") for p in c.split(",") if p]
            old = [(key, _lib.config_get(key)) for key, _ in kv]
            for key, val in kv:
                _lib.config_set(key, int(val))
            nb = lib.osmx_workspace_bytes(alg, B, V, k if topk else 0)
            ws = torch.zeros(nb, dtype=torch.uint8, device=dev)

            def launch(i, st, ws=ws):
                if topk:
                    st_ = lib.osmx_softmax_topk(alg, x[i].data_ptr(), V, B, V, k, vals.data_ptr(), idx.data_ptr(),
                                                ws.data_ptr(), ws.numel(), st)
                else:
                    st_ = lib.osmx_softmax(alg, x[i].data_ptr(), V, y[i].data_ptr(), V, B, V, ws.data_ptr(),
                                           ws.numel(), st)
                assert st_ == 0

            ms, _ = time_rotating(launch, n, a.reps)
            res[c].append(ms)
            for key, val in old:
                _lib.config_set(key, val)
    for c in cfgs:
        ms = statistics.median(res[c])
        gbs = algo_bytes(a.alg, B, V, k) / (ms * 1e-3) / 1e9
        print(f"{a.alg} {B}x{V} [{c or 'default'}]: {ms:.5f} ms ({' '.join(f'{t:.5f}' for t in res[c])})  "
              f"{gbs:.1f} GB/s frac {gbs / peak:.3f}", flush=True)


if __name__ == "__main__":
    main()
