set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -40 > gpurun_out/r2d_pytest.log
./build/ref_unit_tests_b200 > gpurun_out/r2d_refsuite.log 2>&1; echo "refsuite rc=$?" >> gpurun_out/r2d_refsuite.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2d_smoke.log 2>&1
timeout 900 python bench.py --detail-out gpurun_out/r2d_detail.json > gpurun_out/r2d_bench.out 2> gpurun_out/r2d_bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2d_ref.out 2> gpurun_out/r2d_ref.err
tail -3 gpurun_out/r2d_refsuite.log
tail -15 gpurun_out/r2d_pytest.log
tail -c 2200 gpurun_out/r2d_bench.out
tail -c 1500 gpurun_out/r2d_ref.out
