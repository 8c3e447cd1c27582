timeout 300 python tools/c5_sweep.py split_cta=-1 2>&1 | tail -1
timeout 300 python tools/shape_sweep.py --rows 4000 --alg online_fused online --V 32768 131072 --knob shape=0 --reps 9 | grep "^{"
timeout 300 python tools/shape_sweep.py --rows 16384 --alg online_fused --V 131072 --knob shape=0 --reps 9 | grep "^{"
timeout 300 python tools/shape_sweep.py --rows 4000 --alg online --V 5623 100000 177828 1000000 --knob shape=0 --reps 9 | grep "^{"
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
