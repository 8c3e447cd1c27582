# where does the last CTA's combine spend its time
set -x
OSMX_LIB_DIAG=build/tl/libosmx_b200.so python tools/c5_timeline.py > gpurun_out/r2t_timeline.txt 2>&1
cat gpurun_out/r2t_timeline.txt
