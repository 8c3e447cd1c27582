# dyn default + graph-amortized sweep timing: full GPU suite, default bench (sweeps), c5 sweep
set -x
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2y_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2y_pytest.log
timeout 900 python bench.py --detail-out gpurun_out/r2y_detail.json > gpurun_out/r2y_bench.out 2> gpurun_out/r2y_bench.err
python tools/c5_sweep.py split_cta=-1 split_cta=2,tma_cfg=0 > gpurun_out/r2y_c5.txt 2>&1
tail -3 gpurun_out/r2y_pytest.log; tail -c 1800 gpurun_out/r2y_bench.out; cat gpurun_out/r2y_c5.txt
