# One full measurement pass: bench line, launch list, full ncu capture of the headline kernel.
set -x
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --sweep off --e2e off --cpu off > gpurun_out/bench_ncu.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_topk_rows -c 1 -o gpurun_out/prof_c4 python tools/run_op.py --alg online_fused --rows 8192 --V 131072 --reps 1 > /dev/null 2>&1
