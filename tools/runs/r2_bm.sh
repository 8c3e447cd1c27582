# flakiness check: the full GPU suite twice on the final build + smoke
set -x
for i in 1 2; do timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2bm_pytest$i.log 2>&1; echo "pytest$i rc=$?" >> gpurun_out/r2bm_status.txt; done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2bm_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2bm_status.txt
cat gpurun_out/r2bm_status.txt; tail -n 2 gpurun_out/r2bm_pytest1.log gpurun_out/r2bm_pytest2.log; cat gpurun_out/r2bm_smoke.log
