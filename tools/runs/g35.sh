# new cluster rule: defaults across V, plus parity of the staged/cluster paths
for V in 17000 20000 24000 30000 36000 40000 50000 60000 69120 75000 90000 100000 110000 126976 150000 165888 177828; do
  timeout 300 python tools/shape_sweep.py --rows 4000 --alg online safe --V $V --knob cluster_size=0 --reps 9 2>&1 | grep -E "^\{"
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cluster or staged or softmax" 2>&1 | tail -3
