# default cluster layout vs alternatives (cluster size x group width), 4000 rows
for V in 36000 50000 75000 100000 126976 150000; do
  timeout 300 python tools/shape_sweep.py --rows 4000 --alg online safe --V $V --knob cluster_size=0 --reps 7 2>&1 | grep -E "^\{" | sed "s/^/default /"
  for gw in 4 8; do
    timeout 300 python tools/shape_sweep.py --rows 4000 --alg online safe --V $V \
       --set staged_gw=$gw --knob cluster_size=3,4,5,6,7,8,9,10 --reps 7 2>&1 | grep -E "^\{" | sed "s/^/gw$gw /"
  done
done
