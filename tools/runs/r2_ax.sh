# ncu of the two-pass large-k kernel at k = 1000 and k = 33 (4000 x 131072)
set -x
for k in 1000 33; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_topk_large" -c 1 -o /tmp/r2ax_k$k python tools/run_op.py --alg online_fused --rows 4000 --V 131072 --k $k --reps 1 > gpurun_out/r2ax_ncu$k.log 2>&1
ncu -i /tmp/r2ax_k$k.ncu-rep --page details --print-details all > gpurun_out/r2ax_k${k}_details.txt 2>&1
ncu -i /tmp/r2ax_k$k.ncu-rep --page source --csv --print-source sass > gpurun_out/r2ax_k${k}_sass.csv 2>&1
done
python3 tools/ncu_details_summary.py gpurun_out/r2ax_k1000_details.txt gpurun_out/r2ax_k33_details.txt | head -80
