# dyn combine with ordered insertion; C5 timeline; one-row tests; full suite
set -x
timeout 900 python -m pytest tests/test_gpu_onerow.py -q -x -p no:cacheprovider > gpurun_out/r2r_onerow.log 2>&1; echo "rc=$?" >> gpurun_out/r2r_onerow.log
OSMX_LIB_DIAG=build/tl/libosmx_b200.so python tools/c5_timeline.py > gpurun_out/r2r_timeline.txt 2>&1
python tools/c5_sweep.py split_cta=-1 split_cta=4,tma_cfg=0 split_cta=4,tma_cfg=1 split_cta=4,tma_cfg=2 > gpurun_out/r2r_c5.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2r_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2r_pytest.log
tail -3 gpurun_out/r2r_onerow.log; cat gpurun_out/r2r_timeline.txt gpurun_out/r2r_c5.txt; tail -5 gpurun_out/r2r_pytest.log
