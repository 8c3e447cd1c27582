set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/r2a_pytest.log
timeout 300 python bench.py --steps 5 --warmup 3 --sweep off --detail-out gpurun_out/r2a_detail.json > gpurun_out/r2a_bench.out 2> gpurun_out/r2a_bench.err
tail -c 2500 gpurun_out/r2a_bench.out
tail -5 gpurun_out/r2a_pytest.log
