# C5: one-launch wide kernel vs TMA pieces (+fused ticket combine) vs warp pieces; pure-read floor; ncu of the C5 kernels
set -x
./build/c5_lab > gpurun_out/r2n_lab.txt 2>&1
python tools/c5_sweep.py split_cta=-1 split_cta=2 split_cta=3 split_cta=2,split_fuse=1 split_cta=0 split_cta=-1 split_cta=3 > gpurun_out/r2n_c5.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_topk_(tma|combine|wide)" -c 4 -o gpurun_out/r2n_c5_tma python tools/run_op.py --alg online_fused --rows 1 --V 67108864 --reps 2 > gpurun_out/r2n_ncu.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_topk_wide" -c 2 -o gpurun_out/r2n_c5_wide python tools/run_op.py --alg online_fused --rows 1 --V 67108864 --reps 2 --set split_cta=3 >> gpurun_out/r2n_ncu.log 2>&1
cat gpurun_out/r2n_lab.txt gpurun_out/r2n_c5.txt; tail -5 gpurun_out/r2n_ncu.log
