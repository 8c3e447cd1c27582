# c5 one-launch ceiling, CUDA expf accuracy/cost, safe_fused profile, fixed tests
set -x
./build/c5_lab > gpurun_out/r2e_c5lab.txt 2>&1
./build/expf_lab > gpurun_out/r2e_expflab.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "collisions" 2>&1 | tail -5 > gpurun_out/r2e_pytest.log
python tools/run_op.py --alg safe_fused --rows 4000 --V 32768 --reps 7 > gpurun_out/r2e_sf.txt 2>&1
python tools/run_op.py --alg safe_fused --rows 4000 --V 1048576 --reps 3 >> gpurun_out/r2e_sf.txt 2>&1
timeout 300 ncu --set full --clock-control none -k regex:k_topk_rows -c 1 -o gpurun_out/r2e_sf32k python tools/run_op.py --alg safe_fused --rows 4000 --V 32768 --reps 1 > /dev/null 2>&1
cat gpurun_out/r2e_c5lab.txt gpurun_out/r2e_expflab.txt gpurun_out/r2e_sf.txt gpurun_out/r2e_pytest.log
