# large-k pass-A histogram pruned after a 16K-element sample: parity + timing
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "large" > gpurun_out/r2bi_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2bi_pytest.log
for k in 33 100 1000 4096; do python tools/cell_ab.py --alg online_fused --rows 4000 --V 131072 --k $k --cfg "" --rounds 2 --reps 5 >> gpurun_out/r2bi_ab.txt 2>&1; done
python tools/cell_ab.py --alg online_fused --rows 4000 --V 1048576 --k 100 --cfg "" --cfg large_fast=0 --rounds 1 --reps 3 >> gpurun_out/r2bi_ab.txt 2>&1
tail -2 gpurun_out/r2bi_pytest.log; grep online gpurun_out/r2bi_ab.txt
