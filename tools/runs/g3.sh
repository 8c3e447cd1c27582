set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "staged or many_rows or fused_topk_parity or nonfinite or misaligned" > gpurun_out/g3_pytest.log 2>&1; tail -5 gpurun_out/g3_pytest.log
python tools/shape_sweep.py --rows 4000 --alg online safe naive --V 1000 1778 3162 5623 10000 16384 --knob shape=0,4 --reps 7 > gpurun_out/g3_staged.jsonl 2>&1
python tools/shape_sweep.py --rows 4000 --alg online_fused --V 8192 16384 32768 65536 131072 --knob topk_u8=0,1 --reps 7 > gpurun_out/g3_u8.jsonl 2>&1
python tools/shape_sweep.py --rows 65536 --alg online --V 1000 4096 --knob shape=0,4 --reps 5 > gpurun_out/g3_staged_many.jsonl 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_softmax_staged -c 1 -o gpurun_out/g3_staged5623 python tools/run_op.py --alg online --rows 4000 --V 5623 --reps 1 --set shape=4 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_topk_rows -c 1 -o gpurun_out/g3_topk32k_u8 python tools/run_op.py --alg online_fused --rows 4000 --V 32768 --reps 1 > /dev/null 2>&1
