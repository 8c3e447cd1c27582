# full GPU parity + quick timings (+ optional ncu of the C4 kernel with $NCU=1)
python -m pytest tests/ -q -m gpu -x 2>&1 | tail -4
for t in 0 2; do python tools/run_op.py --alg online_fused --rows 16384 --V 131072 --set tma=$t --reps 5; done
for V in 32768 1048576; do for t in 0 2; do python tools/run_op.py --alg online_fused --rows 4000 --V $V --set tma=$t --reps 5; done; done
for V in 1000 10000 100000; do for a in safe online; do python tools/run_op.py --alg $a --rows 4000 --V $V --reps 5; done; done
if [ "$NCU" = "1" ]; then
ncu --set full --import-source on --clock-control none -k regex:k_topk_rows -c 1 -o gpurun_out/prof_rows3 python tools/run_op.py --alg online_fused --rows 4096 --V 131072 --set tma=0 --reps 1 > /dev/null
fi
