for i in 1 2; do
  for d in _ab .; do
    (cd $d && timeout 300 python tools/shape_sweep.py --rows 4000 --alg online --V 3162 5623 10000 17783 31623 100000 --knob shape=0 --reps 9 | grep "^{" | sed "s|^|$d |")
  done
done
(timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_random.py -q -x 2>&1 | tail -2)
