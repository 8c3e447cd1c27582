# synccheck / memcheck over every family after the reconverging barriers in topk_large; large-k parity
set -x
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_run.py > gpurun_out/r2bc_synccheck.txt 2>&1; echo "synccheck rc=$?" >> gpurun_out/r2bc_status.txt
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_run.py > gpurun_out/r2bc_memcheck.txt 2>&1; echo "memcheck rc=$?" >> gpurun_out/r2bc_status.txt
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python tools/sanitize_run.py > gpurun_out/r2bc_racecheck.txt 2>&1; echo "racecheck rc=$?" >> gpurun_out/r2bc_status.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "large" > gpurun_out/r2bc_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2bc_status.txt
for k in 100 1000; do python tools/cell_ab.py --alg online_fused --rows 4000 --V 131072 --k $k --cfg "" --rounds 2 --reps 5 >> gpurun_out/r2bc_ab.txt 2>&1; done
cat gpurun_out/r2bc_status.txt; tail -n 2 gpurun_out/r2bc_synccheck.txt; tail -n 2 gpurun_out/r2bc_memcheck.txt; tail -n 3 gpurun_out/r2bc_racecheck.txt; grep online gpurun_out/r2bc_ab.txt
