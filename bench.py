#!/usr/bin/env python
"""Benchmark of the B200 online-normalizer softmax / fused softmax+TopK.

Headline (BASELINE.json metric "softmax & softmax+Top5 achieved HBM GB/s
(frac of ~8TB/s) and rows/s vs V"), on the configuration the north star
shards across GPUs (configs[3], "C4"): fused online softmax + Top-5 over
65536 rows x V=131072 fp32 per GPU (34.4 GB; rows are independent, so N GPUs
each take their own 65536-row shard -- weak scaling, no collective on the
data path).  A step is one batched launch of the fused kernel over the whole
shard with inputs resident in HBM.  Inputs (34.4 GB) are 270x the 126 MB L2,
so no L2 flush is needed between steps.

Also on the same JSON line (N=1, rank 0):
  e2e           the same metric through the host-buffer C-ABI entry point
                (osmx_softmax_topk_host): pinned host rows -> H2D -> kernel ->
                D2H of the Top-5 per row, all inside the timed region;
  roofline      achieved algorithmic bytes / kernel time vs MEASURED_PEAKS;
  cpu_baseline  the reference's own CPU code (oracle/_ref, built from
                /root/reference/proj/src) on a bounded row sample, all cores;
  sweep         configs[1] (safe vs online softmax, batch 4000, V=10..1M,
                L2 flushed when the working set is < 2x L2) and configs[2]
                (fused vs unfused online->Top-5, batch 4000, V=32K..1M).

`--impl reference` times the reference CPU implementation instead (rank 0
only; other ranks exit 0).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "softmax & softmax+Top5 achieved HBM GB/s (frac of ~8TB/s) and rows/s vs V"
K_TOP = 5


def algo_bytes(alg: str, rows: int, V: int, k: int = K_TOP) -> int:
    """Algorithmic bytes (reference access model counting.hpp:83-86 x 4 B per
    element, 12 B per top-K slot: f32 value + int64 index), SURVEY.md 8d."""
    per = {
        "naive": 12 * V,
        "safe": 16 * V,
        "online": 12 * V,
        "online_fused": 4 * V + 12 * k,
        "online_unfused": 16 * V + 12 * k,
        "safe_unfused": 20 * V + 12 * k,
        "safe_fused": 12 * V + 12 * k,
    }[alg]
    return rows * per


def kernel_name(rows: int, V: int) -> str:
    """The fused top-K kernel the launch layer picks (topk_row_threads /
    run_rows in csrc/topk_impl.cuh) for this shape on a 148-SM B200."""
    if V > 65536 and rows < 3 * 148:
        return "k_topk_rows<32,128,5,kModeFused,4,7,-1> record mode (warp per piece) + combine"
    if V <= 2048 or rows >= 12 * 148 or (rows >= 8 * 148 and V <= 65536):
        if V >= 16384 and rows <= 28 * 148:
            return "k_topk_rows<32,128,5,kModeFused,4,7,-1> (warp per row, register double-buffered)"
        pf = " + bulk L2 prefetch" if V >= 32768 and rows >= 64 * 148 else ""
        return "k_topk_rows<32,256,5,kModeFused,4,4> (warp per row" + pf + ")"
    if rows >= 8 * 148:
        return "k_topk_rows<256,256,5,kModeFused,4,4>"
    if rows >= 2 * 148:
        return "k_topk_rows<128,128,5,kModeFused,4,8>"
    return "k_topk_rows<256,256,5,kModeFused,4,4>"


def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


# ----------------------------------------------------------- clock sampler --

class NvmlClockSampler:
    """SM clock / clock-event reasons sampled every 10 ms through NVML (the
    library nvidia-smi reads) during the timed region -- no process start-up
    inside the window, so short regions still get samples."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4}

    def __init__(self, gpu_index: int):
        import pynvml

        self.nv = pynvml
        pynvml.nvmlInit()
        self.h = pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
        self.smax = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
        self.sm: list[float] = []
        self.mask = 0
        self.stop_ev = threading.Event()
        self.thread = None

    def _run(self):
        nv = self.nv
        while not self.stop_ev.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
                self.mask |= int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:  # noqa: BLE001 -- a failed sample is skipped
                pass
            self.stop_ev.wait(0.01)

    def start(self):
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def stop(self) -> dict:
        self.stop_ev.set()
        if self.thread:
            self.thread.join(timeout=2)
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.smax, "reasons": ["no samples"], "samples": 0}
        reasons = sorted(n for n, b in self.REASONS.items() if self.mask & b)
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.smax, "reasons": reasons,
                "samples": len(self.sm), "source": "nvml"}


def clock_sampler(gpu_index: int):
    """NVML sampler when pynvml is importable, else nvidia-smi -lms."""
    try:
        return NvmlClockSampler(gpu_index)
    except Exception:  # noqa: BLE001 -- no NVML: fall back to the CLI
        return ClockSampler(gpu_index)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "50",
                 "-i", str(self.gpu)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[4:8]):
                if val.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------- reference --

def reference_rate(rows_sample, V: int, k: int, threads: int, repeats: int = 1):
    """Time the reference library (oracle/_ref) on host rows; returns
    (seconds per call (median), kind)."""
    from oracle import oracle as O

    import numpy as np

    lib = O.ref() if O.ref_available() else None
    kind = "reference" if lib is not None else "port"
    x = np.ascontiguousarray(rows_sample, dtype=np.float32)
    rows = x.shape[0]
    v = np.empty((rows, k), np.float32)
    z = np.empty((rows, k), np.int64)
    st = np.empty(rows, np.int32)
    ts = []
    for _ in range(repeats):
        t0 = time.perf_counter()
        if lib is not None:
            lib.osmx_ref_batch(O.OPS["online_softmax_topk"], x.ctypes.data, V, rows, V, k, None, 0, v.ctypes.data,
                               z.ctypes.data, st.ctypes.data, threads)
        else:
            O.port().oracle_batch(O.OPS["online_softmax_topk"], x.ctypes.data, V, rows, V, k, None, 0,
                                  v.ctypes.data, z.ctypes.data, st.ctypes.data, threads)
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts), kind, (v, z)


def host_rows(seed: int, rows: int, V: int):
    """Standard-normal fp32 rows generated on the host (numpy, chunked)."""
    import numpy as np

    rng = np.random.default_rng(seed)
    out = np.empty((rows, V), np.float32)
    step = max(1, (1 << 26) // V)
    for r0 in range(0, rows, step):
        out[r0:r0 + step] = rng.standard_normal((min(step, rows - r0), V), dtype=np.float32)
    return out


def run_reference_arm(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as O

    threads = O.host_threads()
    V, k = args.V, K_TOP
    # size the per-step sample so the whole run stays within ~2-3 minutes
    probe_rows = 64
    xs = host_rows(1234, probe_rows, V)
    t_probe, kind, _ = reference_rate(xs, V, k, threads)
    per_row = t_probe / probe_rows
    total_steps = args.steps + args.warmup
    budget_s = 150.0
    rows_sample = int(max(16, min(args.rows, 8192, budget_s / max(total_steps, 1) / per_row)))
    xs = host_rows(1234, rows_sample, V)
    times = []
    for i in range(total_steps):
        t, kind, _ = reference_rate(xs, V, k, threads)
        if i >= args.warmup:
            times.append(t)
    tot = sum(times)
    gbs = algo_bytes("online_fused", rows_sample, V, k) * len(times) / tot / 1e9
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": round(gbs, 4),
        "unit": "GB/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(tot / len(times) * 1e3, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic standard-normal fp32 rows (numpy), host memory",
        "config": {"workload": "C4 fused online softmax+Top-5 (reference online_softmax_topk, CPU)",
                   "rows": rows_sample, "V": V, "k": k, "rows_per_step_sample": rows_sample},
        "rows_per_s": round(rows_sample * len(times) / tot, 3),
        "elements_per_s": round(rows_sample * V * len(times) / tot, 1),
        "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": threads, "kind": kind,
                         "sample": f"{rows_sample} rows x V={V} per step (bounded sample of C4), "
                                   f"{threads} threads striped like run_batch (bench.cpp:75-90)"},
        "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ ours --

def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rows", type=int, default=65536, help="rows per GPU (weak scaling)")
    ap.add_argument("--V", type=int, default=131072)
    ap.add_argument("--sweep", default="auto", choices=["auto", "on", "off"])
    ap.add_argument("--e2e", default="auto", choices=["auto", "on", "off"])
    ap.add_argument("--cpu", default="auto", choices=["auto", "on", "off"])
    ap.add_argument("--sweep-reps", type=int, default=20)
    ap.add_argument("--detail-out", default=None,
                    help="write the full result (sweeps, V-split, notes) as JSON to this path")
    ap.add_argument("--sweep-only", action="store_true", help="print only the configs[1]/[2]/[4] sweeps (N=1)")
    ap.add_argument("--vsplit", default="auto", choices=["auto", "on", "off"],
                    help="configs[4] across ranks: one 2^26 row split over the N GPUs, NCCL record all-gather "
                         "(auto: when N > 1)")
    args = ap.parse_args()

    if args.impl == "reference":
        run_reference_arm(args)
        return

    import numpy as np
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if args.sweep_only:
        from paper_1805_02867_b200 import _lib

        lib = _lib.load()
        ss = clock_sampler(local)
        ss.start()
        sweep = run_sweeps(lib, _lib, dev, torch.cuda.current_stream(dev).cuda_stream, args.sweep_reps,
                           measured_peaks()["hbm_gbs"])
        sweep["clocks"] = ss.stop()
        print(json.dumps({"metric": METRIC, "sweep": sweep}), flush=True)
        return
    dist = None
    if world > 1 or args.vsplit == "on":
        import torch.distributed as dist

        if not dist.is_initialized():
            if world == 1:  # a one-rank group, so the V-split's collective runs too
                os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
                os.environ.setdefault("MASTER_PORT", "29531")
                dist.init_process_group("nccl", device_id=dev, rank=0, world_size=1)
            else:
                dist.init_process_group("nccl", device_id=dev)

    from paper_1805_02867_b200 import _lib, osmx

    lib = _lib.load()
    rows, V, k = args.rows, args.V, K_TOP
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream

    # ---- synthetic C4 shard, resident in HBM
    g = torch.Generator(device=dev)
    g.manual_seed(1000 + rank)
    x = torch.empty((rows, V), dtype=torch.float32, device=dev)
    x.normal_(generator=g)
    vals = torch.empty((rows, k), dtype=torch.float32, device=dev)
    idx = torch.empty((rows, k), dtype=torch.int64, device=dev)
    alg = _lib.ONLINE_SOFTMAX_FUSED_TOPK
    nb = lib.osmx_workspace_bytes(alg, rows, V, k)
    ws = torch.zeros(max(nb, 256), dtype=torch.uint8, device=dev)

    def step():
        st = lib.osmx_softmax_topk(alg, x.data_ptr(), V, rows, V, k, vals.data_ptr(), idx.data_ptr(),
                                   ws.data_ptr(), ws.numel(), sp)
        if st != 0:
            raise RuntimeError(f"osmx_softmax_topk: {_lib.status_string(st)}")

    for _ in range(args.warmup):
        step()
    osmx.check_status(ws, sp)  # warm-up results are finite rows

    # parity spot check of the bench's own output (outside the timed region)
    parity = None
    if rank == 0:
        from oracle import oracle as O

        sample = list(range(0, rows, max(1, rows // 8)))[:8]
        xs = x[sample].cpu().numpy()
        rv, rz, _ = O.batch("online_softmax_topk", xs, k=k)
        gi = idx[sample].cpu().numpy()
        gv = vals[sample].cpu().numpy()
        parity = {"rows_checked": len(sample), "indices_bit_exact": bool(np.array_equal(gi, rz)),
                  "max_rel_err": float(np.max(np.abs(gv.astype(np.float64) - rv) / rv))}

    # ---- timed region
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = clock_sampler(local)
    sampler.start()
    if isinstance(sampler, ClockSampler):
        time.sleep(0.2)  # nvidia-smi start-up (NVML samples from the first call)
    launches0 = _lib.launch_count()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for i in range(args.steps):
        evs[i][0].record(stream)
        step()
        evs[i][1].record(stream)
    t_end.record(stream)
    torch.cuda.synchronize()
    launches = _lib.launch_count() - launches0
    clocks = sampler.stop()
    if dist is not None:
        dist.barrier()
    elapsed_ms = t_start.elapsed_time(t_end)
    kernel_ms = statistics.mean(a.elapsed_time(b) for a, b in evs)
    if dist is not None:
        t = torch.tensor([elapsed_ms, kernel_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms, kernel_ms = float(t[0]), float(t[1])
    osmx.check_status(ws, sp)

    ms_per_step = elapsed_ms / args.steps
    total_rows = rows * world
    bytes_step = algo_bytes("online_fused", total_rows, V, k)
    value = bytes_step / (ms_per_step * 1e-3) / 1e9
    peaks = measured_peaks()
    bytes_launch = algo_bytes("online_fused", rows, V, k)
    achieved = bytes_launch / (kernel_ms * 1e-3) / 1e9

    result = {
        "metric": METRIC,
        "value": round(value, 2),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic standard-normal fp32 logits (torch normal_ on device)",
        "config": {"workload": "C4 fused online softmax+Top-5 (online_softmax_topk, Alg. 4), rows sharded",
                   "rows_per_gpu": rows, "V": V, "k": k, "parallelism": f"row-shard x{world} (no collective)",
                   "l2": "inputs 34.4 GB/GPU >> 126 MB L2: no flush needed"},
        "rows_per_s": round(total_rows / (ms_per_step * 1e-3), 1),
        "elements_per_s": round(total_rows * V / (ms_per_step * 1e-3), 1),
        "gpu_launches": int(launches),
        "clocks": clocks,
        "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": round(achieved / peaks["hbm_gbs"], 4), "traffic": None,
                     "kernel": kernel_name(rows, V),
                     "algorithmic_bytes_per_launch": bytes_launch,
                     "avg_launch_ms": round(kernel_ms, 4), "peak_source": peaks["source"]},
        "parity": parity,
    }
    # context for frac > 1 (the peak is a read+write copy): the achievable
    # pure-read bandwidth of the same shard, measured by the library's
    # diagnostic read probe (128-bit grid-stride loads, nothing else)
    if rank == 0:
        sink = torch.zeros(1, dtype=torch.float32, device=dev)
        lib.osmx_diag_read_probe(x.data_ptr(), x.numel() * 4, sink.data_ptr(), sp)
        torch.cuda.synchronize()
        ra, rb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ra.record(stream)
        for _ in range(5):
            lib.osmx_diag_read_probe(x.data_ptr(), x.numel() * 4, sink.data_ptr(), sp)
        rb.record(stream)
        rb.synchronize()
        probe = x.numel() * 4 * 5 / (ra.elapsed_time(rb) * 1e-3) / 1e9
        result["roofline"]["read_probe_GBps"] = round(probe, 1)
        result["roofline"]["frac_of_read_probe"] = round(achieved / probe, 4)
        result["roofline"]["read_probe_note"] = ("osmx_diag_read_probe over the same shard, right after the timed "
                                                 "region: the pure-read ceiling (context; 'peak' stays the "
                                                 "MEASURED_PEAKS copy figure)")
    traffic = ROOT / "profiles" / "traffic.json"
    if traffic.exists():
        try:
            tj = json.loads(traffic.read_text()).get("online_fused_c4")
            if tj and V == 131072 and k == K_TOP:  # captured on the C4 row length
                result["roofline"]["traffic"] = int(tj["dram_bytes_per_row"] * rows)
                result["roofline"]["traffic_source"] = tj.get("source")
        except (ValueError, KeyError):
            pass

    # ---- e2e through the host-buffer C-ABI entry point (pinned host rows)
    do_e2e = args.e2e == "on" or (args.e2e == "auto")
    if do_e2e:
        e2e = e2e_measure(lib, _lib, x, idx, rows, V, k, dev, world, dist, local, args.steps)
        if e2e is not None:
            result["e2e"] = e2e

    # ---- CPU baseline (rank 0, N=1)
    if rank == 0 and world == 1 and args.cpu != "off":
        result["cpu_baseline"] = cpu_baseline(x, V, k)

    # ---- sweeps (N=1; configs[1], [2], [4] and the fused projection), after
    # the headline (the tensor-core GEMM's power draw would otherwise throttle
    # the headline's HBM stream); one preallocated arena (run_sweeps)
    if rank == 0 and world == 1 and (args.sweep == "on" or args.sweep == "auto"):
        # x stays allocated: a buffer mapped right after a 34 GB free made the
        # latency-bound top-K ~25% slower (tools/placement_test.py)
        ss = clock_sampler(local)
        ss.start()
        sweep = run_sweeps(lib, _lib, dev, sp, args.sweep_reps, measured_peaks()["hbm_gbs"])
        sweep["clocks"] = ss.stop()
        sweep["c1_parity"] = c1_parity(lib, _lib, dev)
        result["sweep"] = sweep
        torch.cuda.empty_cache()

    # ---- configs[4] across ranks (V-split + NCCL record all-gather)
    if args.vsplit == "on" or (args.vsplit == "auto" and world > 1):
        x = None
        torch.cuda.empty_cache()
        result["vsplit_c5"] = vsplit_measure(dist, dev, world, rank, args.steps, args.warmup)

    if rank == 0:
        emit(result, args.detail_out)
    if dist is not None:
        dist.destroy_process_group()


FINAL_LINE_MAX = 2000  # the driver keeps only the tail of stdout: the headline line must stay short


def sweep_summary(sweep: dict) -> dict:
    """The north-star ratios of the sweeps in a few numbers (the full sweep is
    printed on the line before the headline and written to --detail-out)."""
    out = {}
    sm = [r for r in sweep.get("softmax", []) if r["V"] >= 4096]
    if sm:
        out["online_frac_min_V4K"] = min(r["online"]["frac"] for r in sm)
        out["online_over_safe_stream_min_V4K"] = min(r["online_over_safe_stream"] for r in sm)
        out["online_stream_over_safe_stream_min_V31K"] = min(
            (r["online_stream_over_safe_stream"] for r in sm if r["V"] >= 31623), default=None)
    tk = sweep.get("topk", [])
    if tk:
        out["fused_over_online_unfused_min"] = min(r["fused_over_online_unfused"] for r in tk)
        out["fused_frac_min"] = min(r["online_fused"]["frac"] for r in tk)
    c5 = sweep.get("c5")
    if c5:
        out["c5_fused_ms"] = c5["online_fused"]["ms"]
        out["c5_fused_frac"] = c5["online_fused"]["frac"]
    c1 = sweep.get("c1_parity")
    if c1:
        out["c1_max_rel_err"] = max(c1[f"{a}_max_rel_err"] for a in ("naive", "safe", "online"))
    return out


def emit(result: dict, detail_out: str | None) -> None:
    """Print the detail (sweeps, V-split, long notes) on an earlier line and to
    `detail_out`, then the compact headline JSON line (< FINAL_LINE_MAX bytes)
    as the LAST line of stdout."""
    detail = {k: result[k] for k in ("sweep", "vsplit_c5") if k in result}
    detail["roofline"] = result.get("roofline")
    detail["e2e"] = result.get("e2e")
    detail["cpu_baseline"] = result.get("cpu_baseline")
    if detail_out:
        p = Path(detail_out)
        p.parent.mkdir(parents=True, exist_ok=True)
        p.write_text(json.dumps(result, indent=1))
    print(json.dumps({"detail": detail}), flush=True)
    line = compact_line(result)
    print(json.dumps(line, separators=(",", ":")), flush=True)


def compact_line(result: dict) -> dict:
    keep = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
            "vs_baseline", "dtype", "data", "config", "rows_per_s", "elements_per_s", "gpu_launches")
    line = {k: result[k] for k in keep if k in result}
    c = result.get("clocks") or {}
    line["clocks"] = {k: c.get(k) for k in ("sm_mhz", "sm_max_mhz", "reasons", "samples")}
    r = result.get("roofline") or {}
    line["roofline"] = {k: r[k] for k in ("bound", "achieved", "peak", "unit", "frac", "traffic", "avg_launch_ms",
                                          "read_probe_GBps", "frac_of_read_probe") if k in r}
    e = result.get("e2e")
    if e:
        line["e2e"] = {k: e[k] for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step", "steps",
                                         "ms_per_step", "devices", "consistent") if k in e}
    cb = result.get("cpu_baseline")
    if cb:
        line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample") if k in cb}
    if result.get("parity"):
        p = result["parity"]
        line["parity"] = {"rows": p["rows_checked"], "idx_exact": p["indices_bit_exact"],
                          "max_rel_err": float(f"{p['max_rel_err']:.3g}")}
    if result.get("sweep"):
        line["sweep"] = sweep_summary(result["sweep"])
    if result.get("vsplit_c5"):
        v = result["vsplit_c5"]
        line["vsplit_c5"] = {"ranks": v["ranks"], "ms": v["ms"], "GBps": v["GBps"]}
        if "vsplit_over_single" in v:
            line["vsplit_c5"]["over_single_gpu"] = v["vsplit_over_single"]
    # hard bound: drop the optional context before the contract keys
    for opt in ("sweep", "vsplit_c5", "parity", "elements_per_s"):
        if len(json.dumps(line, separators=(",", ":"))) <= FINAL_LINE_MAX:
            break
        line.pop(opt, None)
    return line


def vsplit_measure(dist, dev, world, rank, steps, warmup) -> dict:
    """configs[4] split across ranks through the C-ABI (osmx_vsplit_softmax_topk):
    each rank owns a 64-byte aligned column slice of one 2^26 row; one call
    = the slice record (one launch) -> ONE ncclAllGather of the fixed-size
    records on the same stream -> the rank-order merge (one launch).  Slices
    rotate over buffer sets covering >= 4 x L2 (inputs cold, like the
    single-GPU c5 cell), the n_sets calls are captured in one CUDA graph,
    CUDA events, max over ranks.  The single-GPU split path over the same
    slices (osmx_softmax_topk, rank 0's view) is timed the same way."""
    import torch

    from paper_1805_02867_b200 import _lib, osmx, shard

    lib = _lib.load()
    V, k = 1 << 26, K_TOP
    c0, c1 = shard.col_range(V, world, rank)
    n = c1 - c0
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    sets = n_rotating_sets(4 * max(n, 1), l2)
    g = torch.Generator(device=dev)
    g.manual_seed(77)
    xs = torch.empty((sets, max(n, 1)), dtype=torch.float32, device=dev).normal_(generator=g)
    comm = osmx.NcclComm.from_torch_distributed()
    vals = torch.empty(k, dtype=torch.float32, device=dev)
    idx = torch.empty(k, dtype=torch.int64, device=dev)
    nb = lib.osmx_vsplit_workspace_bytes(n, k, world)
    ws = torch.zeros(nb, dtype=torch.uint8, device=dev)
    nb1 = lib.osmx_workspace_bytes(5, 1, max(n, 1), k)
    ws1 = torch.zeros(nb1, dtype=torch.uint8, device=dev)

    def vs(i, st):
        assert lib.osmx_vsplit_softmax_topk(xs[i].data_ptr(), n, c0, k, comm.ptr, vals.data_ptr(), idx.data_ptr(),
                                            ws.data_ptr(), nb, st) == 0, osmx.load().osmx_last_nccl_error()

    def single(i, st):
        assert lib.osmx_softmax_topk(5, xs[i].data_ptr(), n, 1, n, k, vals.data_ptr(), idx.data_ptr(),
                                     ws1.data_ptr(), nb1, st) == 0

    def timed(fn):
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            for _ in range(max(warmup, 1)):
                for i in range(sets):
                    fn(i, st.cuda_stream)
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=st):
                for i in range(sets):
                    fn(i, st.cuda_stream)
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            a.record()
            for _ in range(steps):
                gr.replay()
            b.record()
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / (steps * sets)], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t[0])

    ms = timed(vs)
    top1 = int(idx[0].item())
    ms1 = timed(single) if n > 0 else None
    comm.close()
    gbs = algo_bytes("online_fused", 1, V, k) / (ms * 1e-3) / 1e9
    out = {"rows": 1, "V": V, "k": k, "ranks": world, "ms": round(ms, 5), "GBps": round(gbs, 1),
           "top1_index": top1, "n_sets": sets, "api": "osmx_vsplit_softmax_topk (C-ABI, NCCL on the stream)",
           "collective": "one ncclAllGather of fixed-size records per call", "timing": "CUDA graph, max over ranks"}
    if ms1:
        out["slice_single_gpu_ms"] = round(ms1, 5)
        out["vsplit_over_single"] = round(ms / ms1, 3)
    return out


def e2e_measure(lib, _lib, x, dev_idx, rows, V, k, dev, world, dist, local, steps) -> dict:
    """The headline metric through the library's host-buffer row sharder
    (osmx_softmax_topk_host_multi): pinned host rows -> per-device H2D ->
    fused kernel -> D2H of the top-k, one host thread + PCIe link per GPU,
    all inside the timed region.  Rank 0 drives every GPU of the job from one
    process (the C++ caller's view); the other ranks wait at the barrier.
    Wall clock around `steps` calls (each call synchronises)."""
    import ctypes as C

    import numpy as np
    import torch

    # pinned host rows, bounded by host RAM; each device block replicates
    # (a prefix of) rank 0's shard so every block is checkable on device
    try:
        avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    except (ValueError, OSError):
        avail = 64 << 30
    per_dev = max(1, min(rows, int(0.35 * avail / max(world, 1) / (V * 4))))
    res = None
    if int(os.environ.get("RANK", "0")) == 0:
        res = _e2e_rank0(lib, _lib, x, dev_idx, per_dev, V, k, world, steps)
    if dist is not None:
        dist.barrier()
    return res


def _e2e_rank0(lib, _lib, x, dev_idx, per_dev, V, k, world, steps) -> dict:
    import ctypes as C

    import numpy as np
    import torch

    e_rows = per_dev * world
    host = torch.empty((e_rows, V), dtype=torch.float32, pin_memory=True)
    for r in range(world):
        host[r * per_dev:(r + 1) * per_dev].copy_(x[:per_dev])
    hv = torch.empty((e_rows, k), dtype=torch.float32, pin_memory=True)
    hi = torch.empty((e_rows, k), dtype=torch.int64, pin_memory=True)
    bad = C.c_int64(-1)
    alg = _lib.ONLINE_SOFTMAX_FUSED_TOPK
    devs = (C.c_int * world)(*range(world))

    def call():
        st = lib.osmx_softmax_topk_host_multi(alg, host.data_ptr(), e_rows, V, k, hv.data_ptr(), hi.data_ptr(),
                                              devs, world, C.byref(bad))
        if st != 0:
            raise RuntimeError(f"osmx_softmax_topk_host_multi: {_lib.status_string(st)}")

    call()  # warm-up (allocates the per-device staging)
    t0 = time.perf_counter()
    for _ in range(steps):
        call()
    t = (time.perf_counter() - t0) / steps
    # the host path must return what the device-resident launch returned
    ref = dev_idx[:per_dev].cpu().numpy()
    ok = all(bool(np.array_equal(hi.numpy()[r * per_dev:(r + 1) * per_dev], ref)) for r in range(world))
    lib.osmx_host_release()
    gbs = algo_bytes("online_fused", e_rows, V, k) / t / 1e9
    return {"value": round(gbs, 2), "unit": "GB/s", "h2d_bytes_per_step": e_rows * V * 4,
            "d2h_bytes_per_step": e_rows * k * 12, "rows": e_rows, "devices": world, "steps": steps,
            "ms_per_step": round(t * 1e3, 2), "api": "osmx_softmax_topk_host_multi (pinned host buffers)",
            "consistent": ok}


def cpu_baseline(x, V, k) -> dict:
    from oracle import oracle as O

    threads = O.host_threads()
    probe = x[:32].cpu().numpy()
    t, kind, _ = reference_rate(probe, V, k, threads)
    per_row = t / probe.shape[0]
    n = int(max(64, min(x.shape[0], 10.0 / per_row)))
    xs = x[:n].cpu().numpy()
    t, kind, _ = reference_rate(xs, V, k, threads)
    gbs = algo_bytes("online_fused", n, V, k) / t / 1e9
    # single-thread rate on a smaller sample (threads = 1 and all)
    n1 = max(8, n // max(threads, 1))
    t1, _, _ = reference_rate(x[:n1].cpu().numpy(), V, k, 1)
    return {"value": round(gbs, 4), "unit": "GB/s", "cores": threads, "kind": kind,
            "sample": f"{n} of the C4 rows (V={V}), reference online_softmax_topk, {threads} threads",
            "seconds": round(t, 3), "rows_per_s": round(n / t, 2), "elements_per_s": round(n * V / t, 1),
            "single_thread_GBps": round(algo_bytes("online_fused", n1, V, k) / t1 / 1e9, 4),
            "cpu_model": cpu_model()}


def cpu_model() -> str:
    """/proc/cpuinfo model name (osmx_bench.cpp:24-34)."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def c1_parity(lib, _lib, dev) -> dict:
    """configs[0] (C1): online softmax over 4000 x 1000 checked against the
    reference's naive / safe / online softmax on the same rows (the reference
    library itself, oracle/_ref, on the host), max relative error per alg."""
    import numpy as np
    import torch

    from oracle import oracle as O
    from paper_1805_02867_b200 import osmx

    have_ref = O.ref_available()
    xs = O.generate_inputs(1, 4000, 1000) if have_ref else host_rows(1, 4000, 1000)
    xd = torch.from_numpy(np.ascontiguousarray(xs)).to(dev)
    out = {"rows": 4000, "V": 1000, "checker": "reference library (oracle/_ref)" if have_ref else "oracle port",
           "inputs": "reference generate_inputs(seed 1)" if have_ref else "numpy normal (seed 1)"}
    for name in ("naive", "safe", "online"):
        y = osmx.softmax(xd, alg=name).cpu().numpy().astype(np.float64)
        ref, st = O.batch(f"{name}_softmax", xs, impl="ref" if have_ref else "port")
        m = ref > 1e-30
        out[f"{name}_max_rel_err"] = float(np.max(np.abs(y[m] - ref[m]) / ref[m]))
    return out


class RotTimer:
    """Per-launch device time of `launch(i, stream_handle)` over n_sets
    distinct buffer sets launched back to back (set i's inputs were last
    touched n_sets-1 launches ago, so with n_sets * working set >= 4 x L2
    every launch starts with its inputs out of L2).  The launches are
    captured in one CUDA graph (no host launch gaps): the rotation repeated
    until the graph holds >= graph_ms of work (at most 64 launches), so the
    graph's own launch latency (several us) is not charged to a short
    kernel -- with 2 sets of a 4000 x 32K or a 2^26 row it used to add ~4 us
    per launch.  times(reps) replays it, CUDA events on the launching
    stream, and returns the per-launch ms of each replay; callers may
    interleave several timers (rounds) so clock drift hits all alike."""

    def __init__(self, launch, n_sets: int, graph: bool = True, graph_ms: float = 2.0):
        import torch

        self.launch, self.n_sets = launch, n_sets
        s = self.s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for i in range(n_sets):  # warm-up (and first-touch of every set)
                launch(i, s.cuda_stream)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for i in range(n_sets):  # a per-launch estimate to size the graph
                launch(i, s.cuda_stream)
            e1.record(s)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        est = max(e0.elapsed_time(e1) / n_sets, 1e-4)
        rounds = int(max(1, min(64 // n_sets, -(-graph_ms // (est * n_sets)))))
        self.n_launch = rounds * n_sets
        self.g = None
        if graph:
            self.g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.g, stream=s):
                for j in range(self.n_launch):
                    launch(j % n_sets, s.cuda_stream)
            torch.cuda.synchronize()

    def times(self, reps: int) -> list:
        import torch

        ts = []
        s = self.s
        with torch.cuda.stream(s):
            for _ in range(reps):
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(s)
                if self.g is not None:
                    self.g.replay()
                else:
                    for j in range(self.n_launch):
                        self.launch(j % self.n_sets, s.cuda_stream)
                b.record(s)
                b.synchronize()
                ts.append(a.elapsed_time(b) / self.n_launch)
        torch.cuda.synchronize()
        return ts


def time_rotating(launch, n_sets: int, reps: int, graph: bool = True, graph_ms: float = 2.0):
    """RotTimer for one setting: (median ms per launch, min ms)."""
    ts = RotTimer(launch, n_sets, graph, graph_ms).times(reps)
    return statistics.median(ts), min(ts)


def time_interleaved(timers: dict, reps: int, rounds: int = 3) -> dict:
    """Median per-launch ms of several RotTimers measured in `rounds`
    interleaved rounds (each round replays every timer reps/rounds times),
    so a slow stretch of the box hits every setting, not one."""
    per = max(2, -(-reps // rounds))
    ts = {k: [] for k in timers}
    for _ in range(rounds):
        for k, t in timers.items():
            ts[k] += t.times(per)
    return {k: (statistics.median(v), min(v)) for k, v in ts.items()}


def n_rotating_sets(set_bytes: int, l2: int, cap_bytes: int = 48 << 30) -> int:
    """Buffer sets so that the rotation covers >= 4 x L2 (at least 2)."""
    n = max(2, -(-4 * l2 // max(set_bytes, 1)))
    return int(max(2, min(n, cap_bytes // max(set_bytes, 1))))


Vs_all = [10, 18, 32, 56, 100, 178, 316, 562, 1000, 1778, 3162, 5623, 10000, 17783, 31623, 56234, 100000, 177828,
          316228, 562341, 1000000]  # configs[1]: log_spaced_sizes(10, 1e6, 21)
Vt_all = [32768, 65536, 131072, 262144, 524288, 1048576]  # configs[2]


class Arena:
    """One float32 device buffer; take(offset, shape) returns views of it."""

    def __init__(self, n_floats: int, dev):
        import torch

        self.buf = torch.empty(int(n_floats), dtype=torch.float32, device=dev)

    def take(self, off: int, shape):
        n = 1
        for d in shape:
            n *= d
        return self.buf[off:off + n].view(*shape)


def dram_cells() -> dict:
    """Measured DRAM bytes per sweep cell, {(alg, V): bytes per launch set},
    from the newest profiles/dram_cells_r*.json (tools/dram_cells.py: one
    ncu pass over the same cells, L2 flushed before each)."""
    files = sorted((ROOT / "profiles").glob("dram_cells_r*.json"))
    if not files:
        return {}
    try:
        cells = json.loads(files[-1].read_text())["cells"]
    except (ValueError, KeyError):
        return {}
    return {(c["alg"], c["V"]): c["dram_bytes"] for c in cells} | {"_source": files[-1].name}


def add_dram(cell: dict, dram: dict, alg: str, V: int, ms: float, peak: float) -> None:
    """Beside the algorithmic `frac`: the measured DRAM bytes of the cell and
    the DRAM-byte roofline fraction (measured bytes / this run's time / peak)."""
    b = dram.get((alg, V))
    if b:
        cell["dram_bytes"] = int(b)
        cell["dram_frac"] = round(b / (ms * 1e-3) / 1e9 / peak, 3)


def run_sweeps(lib, _lib, dev, sp, reps, peak) -> dict:
    """configs[1]: safe vs online softmax, batch 4000, V = log_spaced(10, 1e6, 21).
    configs[2]: fused online softmax+Top-5 vs unfused online->TopK, batch 4000,
    V = 32K..1M.  Every launch reads inputs that are out of L2: launches
    rotate over >= 2 buffer sets covering >= 4 x L2, captured in one CUDA
    graph and timed with CUDA events (time_rotating); median of `reps`."""
    import torch

    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    B = 4000
    k = K_TOP
    # One arena for every buffer of the sweep, allocated once: the physical
    # mapping of a buffer allocated after large frees can cost the latency-
    # bound fused top-K ~25% (tools/placement_test.py), so all sizes share
    # one mapping instead of each getting a fresh one.
    need = max(max(2 * n_rotating_sets(8 * B * V, l2) * B * V for V in Vs_all),
               max(n_rotating_sets(4 * B * V, l2) * B * V for V in Vt_all), 2 * n_rotating_sets(8 << 26, l2) << 26)
    arena = Arena(need, dev)
    dram = dram_cells()
    out = {"batch": B, "k": k, "timing": "CUDA graph of >= 2 ms of launches over rotating buffer sets "
                                          "(>= 4 x L2, inputs cold in L2), CUDA events, median over 3 "
                                          "rounds interleaving the algorithms of a V; one preallocated "
                                          "arena for all buffers",
           "dram_bytes_source": dram.get("_source"), "softmax": [], "topk": []}
    Vs = Vs_all
    for V in Vs:
        n = n_rotating_sets(8 * B * V, l2)
        x = arena.take(0, (n, B, V)).normal_()
        y = arena.take(n * B * V, (n, B, V))
        row = {"V": V, "n_sets": n}
        # best kernel family per V (auto), and the paper's one-CTA-per-row
        # streaming kernels (shape 2: every pass reads global memory; the
        # safe baseline of the north star, 3 passes / 4 accesses)
        algs = (("naive", _lib.NAIVE_SOFTMAX, 0), ("safe", _lib.SAFE_SOFTMAX, 0), ("online", _lib.ONLINE_SOFTMAX, 0),
                ("safe_stream", _lib.SAFE_SOFTMAX, 2), ("online_stream", _lib.ONLINE_SOFTMAX, 2))
        timers, keep = {}, []
        for name, alg, shape in algs:
            _lib.config_set("shape", shape)  # in force while the graph is captured
            nb = lib.osmx_workspace_bytes(alg, B, V, 0)
            ws = torch.zeros(max(nb, 256), dtype=torch.uint8, device=dev)
            keep.append(ws)

            def launch(i, st, alg=alg, ws=ws):
                lib.osmx_softmax(alg, x[i].data_ptr(), V, y[i].data_ptr(), V, B, V, ws.data_ptr(), ws.numel(), st)

            timers[name] = RotTimer(launch, n)
            _lib.config_set("shape", 0)
        meas = time_interleaved(timers, reps)
        for name, alg, shape in algs:
            ms, ms_min = meas[name]
            gbs = algo_bytes(name.replace("_stream", ""), B, V) / (ms * 1e-3) / 1e9
            row[name] = {"ms": round(ms, 5), "GBps": round(gbs, 1), "frac": round(gbs / peak, 3),
                         "dram_floor_GBps": round(8 * B * V / (ms * 1e-3) / 1e9, 1),
                         "elements_per_s": round(B * V / (ms * 1e-3), 1)}
            add_dram(row[name], dram, name, V, ms, peak)
        row["online_over_safe"] = round(row["safe"]["ms"] / row["online"]["ms"], 3)
        # the paper's comparison: both algorithms in the streaming kernel family
        row["online_stream_over_safe_stream"] = round(row["safe_stream"]["ms"] / row["online_stream"]["ms"], 3)
        row["online_over_safe_stream"] = round(row["safe_stream"]["ms"] / row["online"]["ms"], 3)
        out["softmax"].append(row)
        del timers, keep, x, y
    for V in Vt_all:
        n = n_rotating_sets(4 * B * V, l2)
        x = arena.take(0, (n, B, V)).normal_()
        vals = torch.empty((B, k), dtype=torch.float32, device=dev)
        idx = torch.empty((B, k), dtype=torch.int64, device=dev)
        row = {"V": V, "n_sets": n}
        algs = (("online_fused", _lib.ONLINE_SOFTMAX_FUSED_TOPK, 0),
                ("online_unfused", _lib.ONLINE_SOFTMAX_UNFUSED_TOPK, 0),
                ("safe_unfused", _lib.SAFE_SOFTMAX_UNFUSED_TOPK, 0),
                ("safe_fused", _lib.SAFE_SOFTMAX_FUSED_TOPK, 0),
                ("online_unfused_stream", _lib.ONLINE_SOFTMAX_UNFUSED_TOPK, 2))
        timers, keep = {}, []
        for name, alg, shape in algs:
            _lib.config_set("shape", shape)  # in force while the graph is captured
            nb = lib.osmx_workspace_bytes(alg, B, V, k)
            ws = torch.zeros(max(nb, 256), dtype=torch.uint8, device=dev)
            keep.append(ws)

            def launch(i, st, alg=alg, ws=ws):
                lib.osmx_softmax_topk(alg, x[i].data_ptr(), V, B, V, k, vals.data_ptr(), idx.data_ptr(),
                                      ws.data_ptr(), ws.numel(), st)

            timers[name] = RotTimer(launch, n)
            _lib.config_set("shape", 0)
        meas = time_interleaved(timers, reps)
        for name, alg, shape in algs:
            ms, ms_min = meas[name]
            gbs = algo_bytes(name.replace("_stream", ""), B, V) / (ms * 1e-3) / 1e9
            row[name] = {"ms": round(ms, 5), "GBps": round(gbs, 1), "frac": round(gbs / peak, 3),
                         "rows_per_s": round(B / (ms * 1e-3), 1)}
            add_dram(row[name], dram, name, V, ms, peak)
        del timers, keep
        row["fused_over_online_unfused"] = round(row["online_unfused"]["ms"] / row["online_fused"]["ms"], 3)
        row["fused_over_safe_unfused"] = round(row["safe_unfused"]["ms"] / row["online_fused"]["ms"], 3)
        # unfused pipeline whose softmax stage is the paper's 3-access streaming kernel
        row["fused_over_online_unfused_stream"] = round(row["online_unfused_stream"]["ms"] / row["online_fused"]["ms"],
                                                        3)
        out["topk"].append(row)
        del x
    out["c5"] = run_c5(lib, _lib, dev, reps, peak, l2, arena)
    out["large_k"] = run_large_k(lib, _lib, dev, reps, peak, l2, arena)
    del arena
    torch.cuda.empty_cache()
    out["proj_fused"] = run_proj(dev, reps)
    torch.cuda.empty_cache()
    return out


def run_large_k(lib, _lib, dev, reps, peak, l2, arena) -> dict:
    """k above the register lists (radix select + ordered
    compaction + sort, csrc/topk_large.cu) on the configs[2] row length,
    4000 x 131072, fused online softmax + top-k for k = 5 (reference point),
    33, 100 and 1000 -- algorithmic bytes 4V + 12k per row."""
    import torch

    B, V = 4000, 131072
    n = n_rotating_sets(4 * B * V, l2)
    x = arena.take(0, (n, B, V)).normal_()
    res = {"rows": B, "V": V, "n_sets": n}
    for k in (5, 33, 100, 1000):
        vals = torch.empty((B, k), dtype=torch.float32, device=dev)
        idx = torch.empty((B, k), dtype=torch.int64, device=dev)
        alg = _lib.ONLINE_SOFTMAX_FUSED_TOPK
        nb = lib.osmx_workspace_bytes(alg, B, V, k)
        ws = torch.zeros(max(nb, 256), dtype=torch.uint8, device=dev)

        def launch(i, st, ws=ws, k=k, vals=vals, idx=idx):
            lib.osmx_softmax_topk(alg, x[i].data_ptr(), V, B, V, k, vals.data_ptr(), idx.data_ptr(), ws.data_ptr(),
                                  ws.numel(), st)

        ms, _ = time_rotating(launch, n, reps)
        gbs = algo_bytes("online_fused", B, V, k) / (ms * 1e-3) / 1e9
        res[f"k{k}"] = {"ms": round(ms, 5), "GBps": round(gbs, 1), "frac": round(gbs / peak, 3),
                        "rows_per_s": round(B / (ms * 1e-3), 1)}
        del ws, vals, idx
    del x
    return res


def run_proj(dev, reps) -> dict:
    """the projection fused with the online softmax + top-5
    (osmx_proj_softmax_topk, tcgen05) on an LM-head shape, against cuBLAS
    (torch.mm, bf16 in, fp32 logits out) followed by the fused top-K kernel.
    Tensor-core bound: TFLOP/s vs MEASURED_PEAKS bf16_tflops."""
    import torch

    from paper_1805_02867_b200 import osmx

    p = ROOT / "MEASURED_PEAKS.json"
    pk = json.loads(p.read_text()) if p.exists() else {}
    peak_tf = float(pk.get("bf16_tflops", 2250.0))
    rows, D, V, k = 4096, 4096, 131072, K_TOP
    g = torch.Generator(device=dev)
    g.manual_seed(9)
    h = (torch.randn((rows, D), device=dev, generator=g) / 8).to(torch.bfloat16)
    w = (torch.randn((V, D), device=dev, generator=g) / 8).to(torch.bfloat16)

    def timed(fn):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(max(reps // 2, 3)):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    t_f = timed(lambda: osmx.proj_softmax_topk(h, w, k, check=False))
    z = torch.mm(h, w.t(), out_dtype=torch.float32)
    t_g = timed(lambda: torch.mm(h, w.t(), out_dtype=torch.float32))
    t_t = timed(lambda: osmx.softmax_topk(z, k, check=False))
    vf, zf = osmx.proj_softmax_topk(h, w, k)
    vu, zu = osmx.softmax_topk(z, k)
    same = float((zf == zu).all(dim=1).float().mean())
    flops = 2.0 * rows * V * D
    return {"rows": rows, "D": D, "V": V, "k": k, "dtype": "bf16 in, fp32 accumulate",
            "fused_ms": round(t_f, 4), "fused_TFLOPs": round(flops / t_f / 1e9, 1),
            "fused_frac_bf16_peak": round(flops / t_f / 1e9 / peak_tf, 3), "peak_TFLOPs": peak_tf,
            "unfused_gemm_ms": round(t_g, 4), "unfused_topk_ms": round(t_t, 4),
            "fused_over_unfused": round((t_g + t_t) / t_f, 3), "rows_same_indices_as_unfused": same,
            "logits_bytes_not_written": rows * V * 4}


def run_c5(lib, _lib, dev, reps, peak, l2, arena=None) -> dict:
    """configs[4] on one GPU: a single row of V = 2^26 (256 MB), fused online
    softmax + Top-5 and online softmax, split over CTAs with the (m, d) /
    top-K record combine (the per-GPU leg of the NCCL V-split)."""
    import torch

    V, k = 1 << 26, K_TOP
    n = n_rotating_sets(8 * V, l2)
    if arena is None:
        arena = Arena(2 * n * V, dev)
    x = arena.take(0, (n, V)).normal_()
    y = arena.take(n * V, (n, V))
    vals = torch.empty((1, k), dtype=torch.float32, device=dev)
    idx = torch.empty((1, k), dtype=torch.int64, device=dev)
    res = {"rows": 1, "V": V, "k": k, "n_sets": n}
    for name, alg in (("online_fused", _lib.ONLINE_SOFTMAX_FUSED_TOPK), ("online", _lib.ONLINE_SOFTMAX)):
        topk = name == "online_fused"
        nb = lib.osmx_workspace_bytes(alg, 1, V, k if topk else 0)
        ws = torch.zeros(max(nb, 256), dtype=torch.uint8, device=dev)

        def launch(i, st, alg=alg, ws=ws, topk=topk):
            if topk:
                lib.osmx_softmax_topk(alg, x[i].data_ptr(), V, 1, V, k, vals.data_ptr(), idx.data_ptr(), ws.data_ptr(),
                                      ws.numel(), st)
            else:
                lib.osmx_softmax(alg, x[i].data_ptr(), V, y[i].data_ptr(), V, 1, V, ws.data_ptr(), ws.numel(), st)

        ms, _ = time_rotating(launch, n, reps)
        gbs = algo_bytes(name, 1, V, k) / (ms * 1e-3) / 1e9
        res[name] = {"ms": round(ms, 5), "GBps": round(gbs, 1), "frac": round(gbs / peak, 3),
                     "elements_per_s": round(V / (ms * 1e-3), 1)}
        add_dram(res[name], dram_cells(), "c5_" + name, V, ms, peak)
    del x, y
    return res


if __name__ == "__main__":
    main()
