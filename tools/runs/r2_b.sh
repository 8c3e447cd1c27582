timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -40 > gpurun_out/r2b_pytest.log
./build/ref_unit_tests_b200 > gpurun_out/r2b_refsuite.log 2>&1; echo "refsuite rc=$?" >> gpurun_out/r2b_refsuite.log
tail -3 gpurun_out/r2b_refsuite.log
tail -25 gpurun_out/r2b_pytest.log
