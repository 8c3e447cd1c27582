# interleaved sweep timing: default bench twice (stability of the summary ratios); sanitizer over the new kernels
set -x
for i in 1 2; do start=$(date +%s); timeout 900 python bench.py --detail-out gpurun_out/r2bb_detail$i.json > gpurun_out/r2bb_bench$i.out 2> gpurun_out/r2bb_bench$i.err; echo "bench$i rc=$? secs=$(( $(date +%s) - start ))" >> gpurun_out/r2bb_status.txt; done
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_run.py > gpurun_out/r2bb_memcheck.txt 2>&1; echo "memcheck rc=$?" >> gpurun_out/r2bb_status.txt
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_run.py > gpurun_out/r2bb_synccheck.txt 2>&1; echo "synccheck rc=$?" >> gpurun_out/r2bb_status.txt
cat gpurun_out/r2bb_status.txt; for i in 1 2; do tail -1 gpurun_out/r2bb_bench$i.out | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['sweep'])"; done; tail -3 gpurun_out/r2bb_memcheck.txt gpurun_out/r2bb_synccheck.txt
