set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "topk" > gpurun_out/g16_pytest.log 2>&1; tail -3 gpurun_out/g16_pytest.log
python tools/shape_sweep.py --rows 4000 --alg online_fused --V 32768 65536 131072 --set topk_threads=32 --knob topk_pipe=0,1,2,3 --reps 7 > gpurun_out/g16_a.jsonl 2>&1
python tools/shape_sweep.py --rows 16384 --alg online_fused --V 131072 --set topk_threads=32 --knob topk_pipe=0,1,2,3 --reps 5 > gpurun_out/g16_b.jsonl 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_topk_rows -c 1 -o gpurun_out/g16_pipe32k python tools/run_op.py --alg online_fused --rows 4000 --V 32768 --reps 1 --set topk_pipe=1 --set topk_threads=32 > /dev/null 2>&1
