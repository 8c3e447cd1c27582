# staged layouts after the D >= NG + 2 rule: stress the former failing defaults and forced knobs
set -x
run() { for i in 1 2 3; do OSMX_WATCHDOG=60 timeout 80 python tools/cell_ab.py --alg online --rows 4000 "$@" --rounds 3 --reps 10 > /tmp/as.txt 2>&1; echo "$* run$i rc=$? $(grep -E '^online|Error|Timeout' /tmp/as.txt | head -1 | cut -c1-70)" >> gpurun_out/r2as_status.txt; done; }
run --V 7500 --cfg ""
run --V 8000 --cfg ""
run --V 7000 --cfg ""
run --V 6500 --cfg ""
run --V 10000 --cfg staged_ng=4
run --V 12500 --cfg ""
run --V 10000 --cfg staged_kb=160
cat gpurun_out/r2as_status.txt
