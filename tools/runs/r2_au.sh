# 2-warp groups up to 8K slices: stress 5623-8192 (online, safe, naive) + parity + graph-relaunch test
set -x
run() { for i in 1 2 3; do OSMX_WATCHDOG=60 timeout 80 python tools/cell_ab.py --rows 4000 "$@" --rounds 3 --reps 10 > /tmp/au.txt 2>&1; echo "$* run$i rc=$? $(grep -E '^(online|safe|naive)|Error|Timeout' /tmp/au.txt | head -1 | cut -c1-70)" >> gpurun_out/r2au_status.txt; done; }
run --alg online --V 7000 --cfg ""
run --alg online --V 7500 --cfg ""
run --alg online --V 8000 --cfg ""
run --alg online --V 5623 --cfg ""
run --alg safe --V 7500 --cfg ""
run --alg naive --V 6100 --cfg ""
run --alg online --V 62000 --cfg ""
timeout 900 python -m pytest tests/test_gpu_graph_relaunch.py tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "graph or softmax" > gpurun_out/r2au_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2au_status.txt
cat gpurun_out/r2au_status.txt; tail -3 gpurun_out/r2au_pytest.log
