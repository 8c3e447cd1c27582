# dyn one-row path default (layout 1), two-barrier CTA epilogue; timeline; onerow + full suite; bench
set -x
OSMX_LIB_DIAG=build/tl/libosmx_b200.so python tools/c5_timeline.py > gpurun_out/r2u_timeline.txt 2>&1
python tools/c5_sweep.py split_cta=-1 split_cta=2,tma_cfg=0 split_cta=-1 > gpurun_out/r2u_c5.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2u_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2u_pytest.log
cat gpurun_out/r2u_timeline.txt gpurun_out/r2u_c5.txt; tail -5 gpurun_out/r2u_pytest.log
