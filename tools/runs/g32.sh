# cluster size x group width sweep for the cluster-staged softmax
set -x
for gw in 4 8 16; do
  timeout 600 python tools/shape_sweep.py --rows 4000 --alg online safe --V 24000 50000 100000 126976 177828 \
     --set staged_gw=$gw --knob cluster_size=2,4,6,8,12,16 --reps 7 2>&1 | grep -E "^\{" | sed "s/^/gw$gw /"
done
