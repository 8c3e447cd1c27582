# wide one-launch split (split_cta=3) parity + timing vs TMA pieces; Recip outputs; sweep
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_masked.py tests/test_gpu_fullsize.py -q -x -k "split or masked or c5 or collisions or nonfinite or known" 2>&1 | tail -8 > gpurun_out/r2g_pytest.log
./build/ref_unit_tests_b200 > gpurun_out/r2g_refsuite.log 2>&1; echo "refsuite rc=$?" >> gpurun_out/r2g_refsuite.log
for sc in 2 3; do for rv in "1 67108864" "8 1048576" "64 1048576" "148 1048576" "400 1048576" "128 262144" "444 131072" "700 131072"; do set -- $rv
python tools/run_op.py --alg online_fused --rows $1 --V $2 --reps 15 --set shape=3 --set split_cta=$sc; done; done > gpurun_out/r2g_wide.txt 2>&1
timeout 600 python bench.py --sweep-only --sweep-reps 10 > gpurun_out/r2g_sweep.json 2> gpurun_out/r2g_sweep.err
tail -3 gpurun_out/r2g_refsuite.log
cat gpurun_out/r2g_pytest.log gpurun_out/r2g_wide.txt
python tools/summarize_bench.py gpurun_out/r2g_sweep.json 2>&1 | head -60
