# which ring configurations fail: D = NG + 1 at several (D, NG); 4 stress runs each
set -x
run() { for i in 1 2 3 4; do OSMX_WATCHDOG=60 timeout 80 python tools/cell_ab.py --alg online --rows 4000 "$@" --rounds 3 --reps 10 > /tmp/aq.txt 2>&1; echo "$* run$i rc=$? $(grep -E '^online|Error|Timeout' /tmp/aq.txt | head -1 | cut -c1-70)" >> gpurun_out/r2aq_status.txt; done; }
run --V 7000 --cfg ""
run --V 10000 --cfg staged_ng=4
run --V 10000 --cfg staged_kb=160
run --V 5623 --cfg staged_ng=8
run --V 6000 --cfg staged_ng=7
cat gpurun_out/r2aq_status.txt
