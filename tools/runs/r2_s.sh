# two-lists-per-lane combine; C5 timeline; full suite
set -x
OSMX_LIB_DIAG=build/tl/libosmx_b200.so python tools/c5_timeline.py > gpurun_out/r2s_timeline.txt 2>&1
python tools/c5_sweep.py split_cta=-1 split_cta=4,tma_cfg=0 split_cta=4,tma_cfg=1 split_cta=4,tma_cfg=2 split_cta=2,tma_cfg=1,split_fuse=1 > gpurun_out/r2s_c5.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2s_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2s_pytest.log
cat gpurun_out/r2s_timeline.txt gpurun_out/r2s_c5.txt; tail -5 gpurun_out/r2s_pytest.log
