for V in 177828 196608; do
 for C in 12 16; do for gw in 4 8 16; do
  timeout 300 python tools/shape_sweep.py --rows 4000 --alg online safe --V $V --set cluster_size=$C --set staged_gw=$gw --knob staged_kb=72,100,110,220 --reps 7 2>&1 | grep -E "^\{" | sed "s/^/C$C gw$gw /"
 done; done
done
