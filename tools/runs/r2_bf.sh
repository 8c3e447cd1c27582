# root cause check: the formerly failing layout (D, NG) = (7, 6) with 4-warp groups, now with non-.aligned named
# barriers (diagnostic build: the layout guard is compiled out)
set -x
run() { for i in 1 2 3 4 5 6; do OSMX_LIB_DIAG=build/tl/libosmx_b200.so OSMX_WATCHDOG=60 timeout 80 python tools/cell_ab.py --alg online --rows 4000 "$@" --rounds 3 --reps 10 > /tmp/bf.txt 2>&1; echo "$* run$i rc=$? $(grep -E '^online|Error|Timeout' /tmp/bf.txt | head -1 | cut -c1-70)" >> gpurun_out/r2bf_status.txt; done; }
run --V 7500 --cfg staged_gw=4,staged_ng=6
run --V 10000 --cfg staged_ng=4
cat gpurun_out/r2bf_status.txt
