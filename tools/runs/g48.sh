for gw in 8 16; do
  timeout 300 python tools/shape_sweep.py --rows 4000 --alg online safe --V 177828 196608 --set staged_gw=$gw --set cluster_size=9 --knob staged_kb=220,227 --reps 7 2>&1 | grep -E "^\{" | sed "s/^/gw$gw /"
done
timeout 300 python tools/shape_sweep.py --rows 4000 --alg online safe --V 177828 --knob cluster_size=0 --reps 7 2>&1 | grep -E "^\{" | sed "s/^/default /"
