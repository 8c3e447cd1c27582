# ncu --set full of the final headline kernel (C4 shard, 16384 rows to bound the replay) and the one-row dyn kernel
set -x
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_topk_rows" -c 1 -o /tmp/r2bh_c4 python tools/run_op.py --alg online_fused --rows 16384 --V 131072 --reps 1 > gpurun_out/r2bh_ncu.log 2>&1
ncu -i /tmp/r2bh_c4.ncu-rep --page details --print-details all > gpurun_out/r2bh_c4_details.txt 2>&1
ncu -i /tmp/r2bh_c4.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed > gpurun_out/r2bh_c4_raw.csv 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_topk_tma_dyn" -c 1 -o /tmp/r2bh_c5 python tools/run_op.py --alg online_fused --rows 1 --V 67108864 --reps 1 >> gpurun_out/r2bh_ncu.log 2>&1
ncu -i /tmp/r2bh_c5.ncu-rep --page details --print-details all > gpurun_out/r2bh_c5_details.txt 2>&1
cat gpurun_out/r2bh_c4_raw.csv | tail -2
