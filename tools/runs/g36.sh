for V in 24000 110000 150000 156672 160000 165888 177828; do
  timeout 300 python tools/shape_sweep.py --rows 4000 --alg online safe naive --V $V --knob cluster_size=0 --reps 9 2>&1 | grep -E "^\{"
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -3
