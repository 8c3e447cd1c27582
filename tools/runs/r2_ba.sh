# final verification: full GPU suite, smoke, default bench, reference arm
set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2ba_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2ba_status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2ba_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2ba_status.txt
start=$(date +%s); timeout 900 python bench.py --detail-out gpurun_out/r2ba_detail.json > gpurun_out/r2ba_bench.out 2> gpurun_out/r2ba_bench.err; echo "bench rc=$? secs=$(( $(date +%s) - start ))" >> gpurun_out/r2ba_status.txt
start=$(date +%s); timeout 900 python bench.py --impl reference > gpurun_out/r2ba_ref.out 2> gpurun_out/r2ba_ref.err; echo "ref rc=$? secs=$(( $(date +%s) - start ))" >> gpurun_out/r2ba_status.txt
cat gpurun_out/r2ba_status.txt; tail -3 gpurun_out/r2ba_pytest.log; cat gpurun_out/r2ba_smoke.log; tail -c 1500 gpurun_out/r2ba_bench.out; tail -c 800 gpurun_out/r2ba_ref.out
