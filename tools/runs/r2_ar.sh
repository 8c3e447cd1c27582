# D = NG + 1 with odd NG vs even NG
set -x
run() { for i in 1 2 3 4; do OSMX_WATCHDOG=60 timeout 80 python tools/cell_ab.py --alg online --rows 4000 "$@" --rounds 3 --reps 10 > /tmp/ar.txt 2>&1; echo "$* run$i rc=$? $(grep -E '^online|Error|Timeout' /tmp/ar.txt | head -1 | cut -c1-70)" >> gpurun_out/r2ar_status.txt; done; }
run --V 8000 --cfg staged_ng=5
run --V 6500 --cfg staged_ng=7
run --V 14500 --cfg ""
run --V 12500 --cfg ""
run --V 8000 --cfg staged_ng=4
cat gpurun_out/r2ar_status.txt
