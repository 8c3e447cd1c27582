# One full measurement pass for the round: bench line, launch list of the
# headline, full ncu captures of the headline kernel and the softmax families.
set -x
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/rp_bench.json 2> gpurun_out/rp_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/rp_launches.csv python bench.py --steps 3 --warmup 3 --sweep off --e2e off --cpu off > gpurun_out/rp_bench_ncu.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_topk_rows -c 1 -o gpurun_out/rp_c4 python tools/run_op.py --alg online_fused --rows 8192 --V 131072 --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_topk_rows -c 1 -o gpurun_out/rp_topk32k python tools/run_op.py --alg online_fused --rows 4000 --V 32768 --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_softmax -c 1 -o gpurun_out/rp_sm5623 python tools/run_op.py --alg online --rows 4000 --V 5623 --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_softmax -c 1 -o gpurun_out/rp_sm100k python tools/run_op.py --alg online --rows 4000 --V 100000 --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_softmax -c 1 -o gpurun_out/rp_sm1m python tools/run_op.py --alg online --rows 1000 --V 1000000 --reps 1 > /dev/null 2>&1
