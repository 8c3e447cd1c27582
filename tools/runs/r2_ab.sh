# 1024-thread stream CTAs (safe/online); full-size sweep-cell parity; full suite; default bench
set -x
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2ab_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2ab_pytest.log
timeout 900 python bench.py --detail-out gpurun_out/r2ab_detail.json > gpurun_out/r2ab_bench.out 2> gpurun_out/r2ab_bench.err
tail -3 gpurun_out/r2ab_pytest.log; tail -c 1500 gpurun_out/r2ab_bench.out
