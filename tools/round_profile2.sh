set -x
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/rp3_launches.csv python bench.py --steps 3 --warmup 3 --sweep off --e2e off --cpu off > gpurun_out/rp3_bench_ncu.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_topk_rows -c 1 -o gpurun_out/rp3_c4 python tools/run_op.py --alg online_fused --rows 16384 --V 131072 --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_softmax -c 1 -o gpurun_out/rp3_safe177k python tools/run_op.py --alg safe --rows 4000 --V 177828 --reps 1 > /dev/null 2>&1
