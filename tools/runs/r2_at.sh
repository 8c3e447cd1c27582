# staged ring rule + depth cap; full GPU suite (incl. graph-relaunch stress); default bench with large-k entry
set -x
timeout 2000 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2at_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2at_pytest.log
timeout 900 python bench.py --detail-out gpurun_out/r2at_detail.json > gpurun_out/r2at_bench.out 2> gpurun_out/r2at_bench.err
tail -4 gpurun_out/r2at_pytest.log; tail -c 1500 gpurun_out/r2at_bench.out
