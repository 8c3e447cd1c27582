# staged ring size (shared memory per CTA) vs row length, online and safe (watchdog-bounded)
set -x
for V in 7500 10000 12500 14500 31623 56234; do
OSMX_WATCHDOG=200 timeout 240 python tools/cell_ab.py --alg online --rows 4000 --V $V --cfg "" --cfg staged_kb=120 --cfg staged_kb=140 --cfg staged_kb=160 --cfg staged_kb=180 --cfg staged_kb=200 --rounds 3 --reps 10
done > gpurun_out/r2ad_kb.txt 2>&1
for A in safe naive; do
OSMX_WATCHDOG=100 timeout 120 python tools/cell_ab.py --alg $A --rows 4000 --V 10000 --cfg "" --cfg staged_kb=120 --cfg staged_kb=160 --rounds 3 --reps 10 >> gpurun_out/r2ad_kb.txt 2>&1
done
timeout 300 python -m pytest tests/test_gpu_graph_relaunch.py -q -p no:cacheprovider >> gpurun_out/r2ad_kb.txt 2>&1
grep -E "^(online|safe|naive)|passed|failed" gpurun_out/r2ad_kb.txt
