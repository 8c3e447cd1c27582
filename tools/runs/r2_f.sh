# accurate safe d (double) + out_md outputs; safe fused x-space prefilter
set -x
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/r2f_pytest.log
./build/ref_unit_tests_b200 > gpurun_out/r2f_refsuite.log 2>&1; echo "refsuite rc=$?" >> gpurun_out/r2f_refsuite.log
timeout 600 python bench.py --sweep-only --sweep-reps 10 > gpurun_out/r2f_sweep.json 2> gpurun_out/r2f_sweep.err
tail -3 gpurun_out/r2f_refsuite.log
tail -8 gpurun_out/r2f_pytest.log
python tools/summarize_bench.py gpurun_out/r2f_sweep.json 2>&1 | head -60
