set -x
python tools/run_op.py --alg online_fused --rows 16384 --V 131072 --set tma=0 --reps 5
python tools/run_op.py --alg online_fused --rows 16384 --V 131072 --set tma=2 --reps 5
ncu --set full --import-source on -k regex:k_topk_rows -c 1 -o gpurun_out/prof_rows python tools/run_op.py --alg online_fused --rows 4096 --V 131072 --set tma=0 --reps 1
ncu --set full --import-source on -k regex:k_topk_tma -c 1 -o gpurun_out/prof_tma python tools/run_op.py --alg online_fused --rows 4096 --V 131072 --set tma=2 --reps 1
