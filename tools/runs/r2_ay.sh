# large-k after the shift-based bitonic indexing: timing + parity
set -x
for k in 33 100 1000 4096; do python tools/cell_ab.py --alg online_fused --rows 4000 --V 131072 --k $k --cfg "" --rounds 2 --reps 5 >> gpurun_out/r2ay_ab.txt 2>&1; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "large" > gpurun_out/r2ay_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2ay_pytest.log
grep -E "^online" gpurun_out/r2ay_ab.txt; tail -2 gpurun_out/r2ay_pytest.log
