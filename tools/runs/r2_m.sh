# re-entry baseline: full GPU suite, smoke, default bench
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2m_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2m_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2m_smoke.log 2>&1
timeout 900 python bench.py --detail-out gpurun_out/r2m_detail.json > gpurun_out/r2m_bench.out 2> gpurun_out/r2m_bench.err
tail -4 gpurun_out/r2m_pytest.log; cat gpurun_out/r2m_smoke.log; tail -c 2500 gpurun_out/r2m_bench.out; tail -3 gpurun_out/r2m_bench.err
