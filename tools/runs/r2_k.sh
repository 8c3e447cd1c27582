# butterfly warp top-K merge; 1-warp CTAs default; full GPU suite + c5 A/B + sweep
set -x
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -8 > gpurun_out/r2k_pytest.log
./build/ref_unit_tests_b200 > gpurun_out/r2k_refsuite.log 2>&1; echo "refsuite rc=$?" >> gpurun_out/r2k_refsuite.log
python tools/c5_sweep.py split_fuse=0 split_fuse=1 > gpurun_out/r2k_c5ab.txt 2>&1
timeout 600 python bench.py --sweep-only --sweep-reps 10 > gpurun_out/r2k_sweep.json 2> gpurun_out/r2k_sweep.err
tail -2 gpurun_out/r2k_refsuite.log
cat gpurun_out/r2k_pytest.log gpurun_out/r2k_c5ab.txt
python tools/summarize_bench.py gpurun_out/r2k_sweep.json 2>&1 | head -60
