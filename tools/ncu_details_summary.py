"""Condense an `ncu --page details --print-details all` text dump (made on
the GPU box, where the .ncu-rep stays) into the lines worth keeping under
profiles/: per kernel the speed-of-light block, launch shape, occupancy,
per-SM active-cycle spread, instruction totals and the warp-state table."""
import re
import sys

KEEP = re.compile(r"^\s+(Duration|Elapsed Cycles|SM Active Cycles|DRAM Throughput|Memory Throughput|"
                  r"Compute \(SM\) Throughput|L2 Cache Throughput|Executed Instructions|Issued Warp Per Scheduler|"
                  r"Registers Per Thread|Achieved Occupancy|Theoretical Occupancy|Block Size|Grid Size|Waves Per SM|"
                  r"DRAM Frequency|SM Frequency|Stall [A-Za-z ]+|Selected|One or More Eligible|Dynamic Shared Memory Per Block)\s")
for path in sys.argv[1:]:
    seen = set()
    print(f"## {path}")
    for line in open(path):
        if line.startswith("  void ") or line.startswith("  [") and "(" in line:
            print(line.rstrip()[:160])
            seen = set()
            continue
        m = KEEP.match(line)
        if m:
            key = " ".join(line.split()[:-1])
            if key in seen and not key.startswith("SM Active Cycles"):
                continue
            seen.add(key)
            print("   " + " ".join(line.split()))
