# staged online softmax layouts at 5.6K-17.8K (same box A/B); ncu launch list of the headline bench
set -x
for V in 5623 10000 17783; do
python tools/cell_ab.py --alg online --rows 4000 --V $V --cfg "" --cfg staged_gw=2 --cfg staged_gw=8 --cfg staged_ng=2 --cfg staged_ng=4 --cfg staged_ng=6 --cfg staged_kb=160 --rounds 3 --reps 10
done > gpurun_out/r2ac_staged.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2ac_launches.csv python bench.py --sweep off --cpu off --e2e off --steps 3 --warmup 3 > gpurun_out/r2ac_ncu_bench.log 2>&1
cat gpurun_out/r2ac_staged.txt; tail -3 gpurun_out/r2ac_launches.csv | cut -c1-300
