# staged edges prefetched before the slot wait; large-k fast vs radix+CUB; stress; parity
set -x
python tools/cell_ab.py --alg online --rows 4000 --V 5623 --cfg "" --cfg staged_gw=4,staged_ng=3 --rounds 3 --reps 10 > gpurun_out/r2av_ab.txt 2>&1
python tools/cell_ab.py --alg online --rows 4000 --V 3162 --cfg "" --rounds 3 --reps 10 >> gpurun_out/r2av_ab.txt 2>&1
python tools/cell_ab.py --alg online --rows 4000 --V 7500 --cfg "" --rounds 3 --reps 10 >> gpurun_out/r2av_ab.txt 2>&1
for k in 33 100 1000; do python tools/cell_ab.py --alg online_fused --rows 4000 --V 131072 --k $k --cfg "" --cfg large_fast=0 --rounds 2 --reps 5 >> gpurun_out/r2av_ab.txt 2>&1; done
python tools/cell_ab.py --alg online_fused --rows 4000 --V 32768 --k 100 --cfg "" --cfg large_fast=0 --rounds 2 --reps 5 >> gpurun_out/r2av_ab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_graph_relaunch.py tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "graph or softmax or nonfinite or large" > gpurun_out/r2av_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2av_pytest.log
cat gpurun_out/r2av_ab.txt | grep -E "^(online|safe)"; tail -2 gpurun_out/r2av_pytest.log
