for g in 32 128 256; do python tools/run_op.py --alg online_fused --rows 65536 --V 131072 --set tma=0 --set topk_threads=$g --reps 3; done
for g in 32 128 256; do python tools/run_op.py --alg online_fused --rows 16384 --V 131072 --set tma=0 --set topk_threads=$g --reps 5; done
for g in 32 128 256 512; do python tools/run_op.py --alg online_fused --rows 4000 --V 32768 --set tma=0 --set topk_threads=$g --reps 5; done
for g in 128 256 512; do python tools/run_op.py --alg online_fused --rows 4000 --V 1048576 --set tma=0 --set topk_threads=$g --reps 5; done
