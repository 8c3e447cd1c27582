# A/B: pre-FFMA2 build (_ab) vs current, same box, alternating
for i in 1 2; do
  for d in _ab .; do
    (cd $d && timeout 300 python tools/shape_sweep.py --rows 65536 --alg online_fused --V 131072 --knob shape=0 --reps 5 | grep "^{" | sed "s|^|$d |")
    (cd $d && timeout 300 python tools/shape_sweep.py --rows 4000 --alg online_fused --V 32768 --knob shape=0 --reps 9 | grep "^{" | sed "s|^|$d |")
  done
done
