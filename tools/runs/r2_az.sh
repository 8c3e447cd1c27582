# large-k with the candidate trim: timing + parity (all large-k tests, one-row, parity suite subset)
set -x
for k in 33 100 1000 4096; do python tools/cell_ab.py --alg online_fused --rows 4000 --V 131072 --k $k --cfg "" --rounds 2 --reps 5 >> gpurun_out/r2az_ab.txt 2>&1; done
python tools/cell_ab.py --alg online_fused --rows 4000 --V 32768 --k 100 --cfg "" --rounds 2 --reps 5 >> gpurun_out/r2az_ab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -q -x -p no:cacheprovider -k "large or topk" > gpurun_out/r2az_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2az_pytest.log
grep -E "^online" gpurun_out/r2az_ab.txt; tail -2 gpurun_out/r2az_pytest.log
