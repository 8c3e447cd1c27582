"""Summarise an ncu report: key metrics + SASS opcode histogram + top stall lines."""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "lts__t_bytes.sum", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__cycles_elapsed.avg.per_second"]
for r in rows[2:]:
    name = r[h.index("Kernel Name")][:90]
    print("==", name)
    for w in want:
        if w in h:
            i = h.index(w)
            print(f"   {w:60s} {r[i]:>14} {units[i]}")
    stalls = [(h[i], r[i]) for i in range(len(h)) if h[i].startswith("smsp__average_warp_latency_issue_stalled_") and h[i].endswith(".ratio")]
    tot = sum(float(v) for _, v in stalls if v.replace('.', '', 1).isdigit())
    top = sorted(((float(v), n) for n, v in stalls if v.replace('.', '', 1).isdigit()), reverse=True)[:6]
    print("   stall cycles/issued instr:", ", ".join(f"{n.split('stalled_')[1].replace('.ratio','')}={v:.2f}" for v, n in top))
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
lines = list(csv.reader(io.StringIO(sass)))
hdr = lines[1]
ie = hdr.index("Instructions Executed")
ss = hdr.index("Warp Stall Sampling (All Samples)")
op = collections.Counter(); st = collections.Counter()
for r in lines[2:]:
    if len(r) > ie and r[ie].isdigit():
        t = r[1].split()
        o = t[1] if t[0].startswith("@") else t[0]
        op[o.split(".")[0]] += int(r[ie])
        st[o.split(".")[0]] += int(r[ss] or 0)
tot = sum(op.values())
print("   warp instr:", tot, " top:", ", ".join(f"{k}={v/tot:.1%}" for k, v in op.most_common(14)))
tots = sum(st.values()) or 1
print("   stall samples by opcode:", ", ".join(f"{k}={v/tots:.1%}" for k, v in st.most_common(10)))
