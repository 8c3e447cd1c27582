for r in 300 444 600 1000; do
  timeout 300 python tools/shape_sweep.py --rows $r --alg online_fused --V 131072 1048576 --knob shape=0,3 --reps 7 2>&1 | grep -E "^\{" | sed "s/^/rows$r /"
done
