# fused (ticket) split combine in the TMA piece kernel; 1-warp CTAs for one-wave top-K
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_masked.py tests/test_gpu_fullsize.py tests/test_gpu_vsplit_nccl.py -q -x -k "split or masked or c5 or nonfinite or vsplit or large_k or many_rows" 2>&1 | tail -8 > gpurun_out/r2i_pytest.log
python tools/c5_sweep.py split_fuse=0 split_fuse=1 split_cta=3 > gpurun_out/r2i_c5ab.txt 2>&1
for b in 128 32; do for V in 16384 32768 65536 131072; do python tools/run_op.py --alg online_fused --rows 4000 --V $V --reps 21 --set topk_block=$b; done; done > gpurun_out/r2i_block.txt 2>&1
for rv in "8 1048576" "64 1048576" "148 1048576" "400 1048576" "128 262144" "444 131072" "700 131072"; do set -- $rv
for f in 0 1; do python tools/run_op.py --alg online_fused --rows $1 --V $2 --reps 15 --set split_fuse=$f; done; done > gpurun_out/r2i_fuse.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2i_c5_launches.csv python tools/c5_probe.py > /dev/null 2>&1
cat gpurun_out/r2i_pytest.log gpurun_out/r2i_c5ab.txt gpurun_out/r2i_block.txt gpurun_out/r2i_fuse.txt
grep -E "k_topk" gpurun_out/r2i_c5_launches.csv | cut -c1-60,200-400 | head
