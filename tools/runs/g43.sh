timeout 300 python tools/c5_sweep.py split_cta=-1 split_cta=0 2>&1 | tail -2
timeout 300 python tools/shape_sweep.py --rows 4000 --alg online_fused --V 32768 131072 --knob tma=0,2 --reps 7 | grep "^{"
timeout 300 python tools/shape_sweep.py --rows 1 --alg online_fused --V 1048576 4194304 --knob split_cta=0,2 --reps 9 | grep "^{"
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "topk or split" 2>&1 | tail -2
