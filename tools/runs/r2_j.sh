# why is the split combine ~11 us?  full ncu of the separate combine and the fused piece kernel
set -x
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_topk_combine_cta -c 1 -o gpurun_out/r2j_comb python tools/c5_probe.py split_fuse=0 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_topk_tma -c 1 -o gpurun_out/r2j_tmaf python tools/c5_probe.py split_fuse=1 > /dev/null 2>&1
ls -la gpurun_out/r2j*
