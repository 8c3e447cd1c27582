timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/r2c_pytest.log
./build/ref_unit_tests_b200 > gpurun_out/r2c_refsuite.log 2>&1; echo "refsuite rc=$?" >> gpurun_out/r2c_refsuite.log
timeout 600 python bench.py --sweep-only --sweep-reps 10 > gpurun_out/r2c_sweep.json 2> gpurun_out/r2c_sweep.err
tail -12 gpurun_out/r2c_refsuite.log
tail -15 gpurun_out/r2c_pytest.log
python tools/summarize_bench.py gpurun_out/r2c_sweep.json 2>&1 | head -60
