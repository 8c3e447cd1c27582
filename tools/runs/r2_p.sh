# ncu of the lean C5 piece kernel (tma_cfg 0 and 1); reports summarised on the box (size cap)
set -x
for c in 0 1; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_topk_(tma|combine)" -c 2 -o /tmp/r2p_c5_cfg$c python tools/run_op.py --alg online_fused --rows 1 --V 67108864 --reps 1 --set tma_cfg=$c > gpurun_out/r2p_ncu$c.log 2>&1
ncu -i /tmp/r2p_c5_cfg$c.ncu-rep --page details --print-details all > gpurun_out/r2p_cfg${c}_details.txt 2>&1
ncu -i /tmp/r2p_c5_cfg$c.ncu-rep --page source --csv --print-source sass -k regex:k_topk_tma > gpurun_out/r2p_cfg${c}_sass.csv 2>&1
done
ls -la gpurun_out
