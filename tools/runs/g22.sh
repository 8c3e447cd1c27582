set -x
timeout 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/g22_pytest.log 2>&1; tail -3 gpurun_out/g22_pytest.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/c5_probe.py 2>/dev/null | grep -E "gpu__time" | python3 -c "
import csv,sys
for r in csv.reader(sys.stdin): print(r[4][:60], r[-1])
"
timeout 900 python bench.py --sweep-only > gpurun_out/g22_sweep.json 2> gpurun_out/g22_sweep.err
