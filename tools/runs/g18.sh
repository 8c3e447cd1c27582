set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -q -m gpu -x -k "topk or golden" > gpurun_out/g18_pytest.log 2>&1; tail -3 gpurun_out/g18_pytest.log
python tools/event_cost.py
python tools/event_cost.py topk_threads=32 topk_pipe=3
python tools/shape_sweep.py --rows 65536 --alg online_fused --V 131072 --knob topk_pipe=0,1,3 --reps 5
ncu --set full --import-source on --clock-control none -k regex:k_topk_rows -c 1 -o gpurun_out/g18_u8 python tools/run_op.py --alg online_fused --rows 4000 --V 32768 --reps 1 > /dev/null 2>&1
