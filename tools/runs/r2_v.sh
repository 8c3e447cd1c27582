set -x
OSMX_LIB_DIAG=build/tl/libosmx_b200.so python tools/c5_timeline.py > gpurun_out/r2v_timeline.txt 2>&1
cat gpurun_out/r2v_timeline.txt
