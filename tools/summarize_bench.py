"""Print the headline and the sweeps of a bench.py JSON line."""
import json
import sys

txt = open(sys.argv[1]).read().strip()
try:
    d = json.loads(txt)  # a --detail-out file (one pretty-printed object)
except json.JSONDecodeError:
    d = json.loads(txt.splitlines()[-1])
if "roofline" in d:
    print({k: d.get(k) for k in ("value", "ms_per_step", "gpu_launches")}, "clocks", d.get("clocks"))
    print("roofline", {k: d["roofline"].get(k) for k in ("achieved", "peak", "frac", "traffic")})
if "e2e" in d:
    print("e2e", d["e2e"]["value"], d["e2e"].get("consistent"))
if "cpu_baseline" in d:
    print("cpu", d["cpu_baseline"]["value"], d["cpu_baseline"]["cores"])
sw = d.get("sweep")
if sw:
    print(f"{'V':>8} {'naive':>9} {'safe':>9} {'online':>9} {'on_frac':>8} {'on_dram':>8} {'on/safe':>7} "
          f"{'safe_str':>9} {'on_str':>9} {'str/str':>7} {'on/s_str':>8}")
    for r in sw["softmax"]:
        print(f"{r['V']:>8} {r.get('naive', {}).get('ms', 0):>9} {r['safe']['ms']:>9} {r['online']['ms']:>9} "
              f"{r['online']['frac']:>8} {r['online']['dram_floor_GBps']:>8} {r['online_over_safe']:>7} "
              f"{r.get('safe_stream', {}).get('ms', 0):>9} {r.get('online_stream', {}).get('ms', 0):>9} "
              f"{r.get('online_stream_over_safe_stream', 0):>7} {r.get('online_over_safe_stream', 0):>8}")
    print(f"{'V':>8} {'fused':>9} {'frac':>6} {'unfused':>9} {'ratio':>6} {'safe_unf':>9} {'ratio':>6} "
          f"{'unf_str':>9} {'ratio':>6}")
    for r in sw["topk"]:
        print(f"{r['V']:>8} {r['online_fused']['ms']:>9} {r['online_fused']['frac']:>6} {r['online_unfused']['ms']:>9} "
              f"{r['fused_over_online_unfused']:>6} {r['safe_unfused']['ms']:>9} {r['fused_over_safe_unfused']:>6} "
              f"{r.get('online_unfused_stream', {}).get('ms', 0):>9} {r.get('fused_over_online_unfused_stream', 0):>6}"
              f"  safe_fused {r.get('safe_fused', {}).get('ms', 0)}")
    if "c5" in sw:
        print("c5", json.dumps(sw["c5"]))
    if "c1_parity" in sw:
        print("c1", json.dumps(sw["c1_parity"]))
    if "proj_fused" in sw:
        print("proj", json.dumps(sw["proj_fused"]))
