# REDUX group_merge everywhere; one-row TMA over dynamic chunks (split_cta=4)
set -x
timeout 900 python -m pytest tests/test_gpu_onerow.py -q -x -p no:cacheprovider > gpurun_out/r2q_onerow.log 2>&1; echo "rc=$?" >> gpurun_out/r2q_onerow.log
python tools/c5_sweep.py split_cta=-1 split_cta=4,tma_cfg=0 split_cta=4,tma_cfg=1 split_cta=4,tma_cfg=2 split_cta=2,tma_cfg=1 split_cta=4,tma_cfg=1 > gpurun_out/r2q_c5.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2q_pytest.log
tail -15 gpurun_out/r2q_onerow.log; cat gpurun_out/r2q_c5.txt; tail -15 gpurun_out/r2q_pytest.log
