# lean L2Acc raise / FADD2 sums / one-vote select; TMA ring layouts for C5
set -x
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2o_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2o_pytest.log
python tools/c5_sweep.py tma_cfg=0 tma_cfg=1 tma_cfg=2 tma_cfg=0,split_fuse=1 tma_cfg=1,split_fuse=1 tma_cfg=2,split_fuse=1 split_cta=3 tma_cfg=0 > gpurun_out/r2o_c5.txt 2>&1
timeout 600 python bench.py --sweep-only --sweep-reps 10 > gpurun_out/r2o_sweep.json 2> gpurun_out/r2o_sweep.err
timeout 300 python bench.py --sweep off --cpu off --e2e off --steps 10 > gpurun_out/r2o_bench.out 2>&1
tail -4 gpurun_out/r2o_pytest.log; cat gpurun_out/r2o_c5.txt; tail -c 600 gpurun_out/r2o_bench.out
python tools/summarize_bench.py gpurun_out/r2o_sweep.json 2>&1 | tail -32
