# final: full GPU suite, smoke, default bench
set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2bg_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2bg_status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2bg_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2bg_status.txt
start=$(date +%s); timeout 900 python bench.py --detail-out gpurun_out/r2bg_detail.json > gpurun_out/r2bg_bench.out 2> gpurun_out/r2bg_bench.err; echo "bench rc=$? secs=$(( $(date +%s) - start ))" >> gpurun_out/r2bg_status.txt
cat gpurun_out/r2bg_status.txt; tail -3 gpurun_out/r2bg_pytest.log; cat gpurun_out/r2bg_smoke.log; tail -c 1700 gpurun_out/r2bg_bench.out
