# A/B: md_group_reduce as max + rescale + sum (.) vs merge tree (_ab)
for i in 1 2; do
  for d in _ab .; do
    (cd $d && timeout 300 python tools/shape_sweep.py --rows 4000 --alg online safe --V 1000 3162 5623 10000 17783 56234 177828 --knob shape=0 --reps 9 | grep "^{" | sed "s|^|$d |")
    (cd $d && timeout 300 python tools/shape_sweep.py --rows 4000 --alg online_fused --V 2048 8192 32768 --knob shape=0 --reps 9 | grep "^{" | sed "s|^|$d |")
  done
done
(timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2)
