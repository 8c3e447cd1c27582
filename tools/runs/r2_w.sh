# ncu of the one-row dyn kernel (layout 1) + 4000 x 32K / 16K fused top-K; summaries only (size cap)
set -x
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_topk_tma_dyn" -c 1 -o /tmp/r2w_dyn python tools/run_op.py --alg online_fused --rows 1 --V 67108864 --reps 1 > gpurun_out/r2w_ncu.log 2>&1
ncu -i /tmp/r2w_dyn.ncu-rep --page details --print-details all > gpurun_out/r2w_dyn_details.txt 2>&1
ncu -i /tmp/r2w_dyn.ncu-rep --page source --csv --print-source sass > gpurun_out/r2w_dyn_sass.csv 2>&1
for V in 32768 16384; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_topk_rows" -c 1 -o /tmp/r2w_rows$V python tools/run_op.py --alg online_fused --rows 4000 --V $V --reps 1 >> gpurun_out/r2w_ncu.log 2>&1
ncu -i /tmp/r2w_rows$V.ncu-rep --page details --print-details all > gpurun_out/r2w_rows${V}_details.txt 2>&1
ncu -i /tmp/r2w_rows$V.ncu-rep --page source --csv --print-source sass > gpurun_out/r2w_rows${V}_sass.csv 2>&1
done
ls -la gpurun_out
