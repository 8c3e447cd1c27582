# NCCL V-split tests; c5 A/B (TMA pieces vs wide) with cold buffers; launch list + ncu of the wide kernel
set -x
timeout 600 python -m pytest tests/test_gpu_vsplit_nccl.py -q -x 2>&1 | tail -15 > gpurun_out/r2h_vsplit.log
python tools/c5_sweep.py split_cta=2 split_cta=3 shape=3,split_cta=3 > gpurun_out/r2h_c5ab.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/r2h_c5_launches.csv python tools/c5_probe.py > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/r2h_c5w_launches.csv python tools/c5_probe.py split_cta=3 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_topk_wide -c 1 -o gpurun_out/r2h_wide python tools/c5_probe.py split_cta=3 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_topk_tma -c 1 -o gpurun_out/r2h_tma python tools/c5_probe.py > /dev/null 2>&1
cat gpurun_out/r2h_vsplit.log gpurun_out/r2h_c5ab.txt
grep -E "k_topk|k_softmax" gpurun_out/r2h_c5_launches.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | cut -c1-160 | head -20
grep -E "k_topk|k_softmax" gpurun_out/r2h_c5w_launches.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | cut -c1-160 | head -20
