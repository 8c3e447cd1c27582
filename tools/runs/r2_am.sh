# staged softmax without cp.async edges: repeat the (D=7, NG=6) V=7500 stress; parity of the staged family
set -x
for i in 1 2 3 4 5 6; do
OSMX_WATCHDOG=80 timeout 100 python tools/cell_ab.py --alg online --rows 4000 --V 7500 --cfg "" --rounds 3 --reps 10 > /tmp/am.txt 2>&1; echo "run$i rc=$? $(grep -E '^online' /tmp/am.txt | cut -c1-50)" >> gpurun_out/r2am_status.txt
done
OSMX_WATCHDOG=80 timeout 100 python tools/cell_ab.py --alg safe --rows 4000 --V 7500 --cfg "" --cfg staged_kb=120 --rounds 3 --reps 10 > /tmp/am.txt 2>&1; echo "safe rc=$? $(grep -E '^safe' /tmp/am.txt | cut -c1-50)" >> gpurun_out/r2am_status.txt
OSMX_WATCHDOG=80 timeout 100 python tools/cell_ab.py --alg naive --rows 4000 --V 7501 --cfg "" --rounds 3 --reps 10 > /tmp/am.txt 2>&1; echo "naive7501 rc=$? $(grep -E '^naive' /tmp/am.txt | cut -c1-50)" >> gpurun_out/r2am_status.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_graph_relaunch.py -q -x -p no:cacheprovider -k "softmax or nonfinite or graph or golden or large_k" > gpurun_out/r2am_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2am_status.txt
cat gpurun_out/r2am_status.txt; tail -3 gpurun_out/r2am_pytest.log
