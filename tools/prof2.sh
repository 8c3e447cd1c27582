python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "topk" 2>&1 | tail -3
for t in 0 2; do python tools/run_op.py --alg online_fused --rows 16384 --V 131072 --set tma=$t --reps 5; done
for V in 32768 1048576; do for t in 0 2; do python tools/run_op.py --alg online_fused --rows 4000 --V $V --set tma=$t --reps 5; done; done
ncu --set full --import-source on --clock-control none -k regex:k_topk_rows -c 1 -o gpurun_out/prof_rows2 python tools/run_op.py --alg online_fused --rows 4096 --V 131072 --set tma=0 --reps 1 > /dev/null
ncu --set full --import-source on --clock-control none -k regex:k_topk_tma -c 1 -o gpurun_out/prof_tma2 python tools/run_op.py --alg online_fused --rows 4096 --V 131072 --set tma=2 --reps 1 > /dev/null
