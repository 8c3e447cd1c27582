# staged V=7500 failure rate: NG=5 (D=7) vs default NG=6, 6 runs each, interleaved; failure text kept
set -x
for i in 1 2 3 4 5 6; do
for c in "staged_ng=5" ""; do
OSMX_WATCHDOG=80 timeout 100 python tools/cell_ab.py --alg online --rows 4000 --V 7500 --cfg "$c" --rounds 3 --reps 10 > /tmp/an.txt 2>&1; rc=$?
echo "run$i [$c] rc=$rc $(grep -E '^online|Error|Timeout' /tmp/an.txt | head -2 | cut -c1-80 | tr '\n' ' ')" >> gpurun_out/r2an_status.txt
done; done
cat gpurun_out/r2an_status.txt
