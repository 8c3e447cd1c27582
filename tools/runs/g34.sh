# cluster sizes that pack 18-SM GPCs (2,3,6,9) vs others, x group width, 4000 rows
for V in 20000 30000 40000 60000 90000 110000 140000 177828 196608; do
  timeout 300 python tools/shape_sweep.py --rows 4000 --alg online safe --V $V --knob cluster_size=0 --reps 7 2>&1 | grep -E "^\{" | sed "s/^/default /"
  for gw in 4 8; do
    timeout 300 python tools/shape_sweep.py --rows 4000 --alg online safe --V $V \
       --set staged_gw=$gw --knob cluster_size=2,3,4,6,9,12,16 --reps 7 2>&1 | grep -E "^\{" | sed "s/^/gw$gw /"
  done
done
