# round-1 session-2 experiments: L2 bulk prefetch, new rotating timing, ncu of the weak shapes
set -x
python tools/shape_sweep.py --rows 4000 --alg online_fused --V 32768 65536 131072 --knob l2_prefetch=0,1,2,4,8 --reps 7 > gpurun_out/g2_topk_pf.jsonl 2>&1
python tools/shape_sweep.py --rows 16384 --alg online_fused --V 131072 --knob l2_prefetch=0,2,4 --reps 5 > gpurun_out/g2_topk_c4_pf.jsonl 2>&1
python tools/shape_sweep.py --rows 4000 --alg online safe --V 1000 1778 3162 5623 10000 17783 31623 100000 --knob l2_prefetch=0,2,4 --reps 7 > gpurun_out/g2_sm_pf.jsonl 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_topk_rows -c 1 -o gpurun_out/g2_topk32k python tools/run_op.py --alg online_fused --rows 4000 --V 32768 --reps 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_softmax -c 1 -o gpurun_out/g2_sm5623 python tools/run_op.py --alg online --rows 4000 --V 5623 --reps 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_softmax -c 1 -o gpurun_out/g2_sm10000 python tools/run_op.py --alg online --rows 4000 --V 10000 --reps 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_softmax -c 1 -o gpurun_out/g2_sm3162 python tools/run_op.py --alg online --rows 4000 --V 3162 --reps 1 > /dev/null 2>&1
timeout 900 python bench.py --steps 20 --e2e off --cpu off > gpurun_out/g2_bench.json 2> gpurun_out/g2_bench.err
tail -c 300 gpurun_out/g2_bench.json
