for r in 128 256 400; do
  timeout 300 python tools/shape_sweep.py --rows $r --alg online_fused --V 262144 1048576 --knob split_cta=0,2 --reps 7 2>&1 | grep -E "^\{" | sed "s/^/rows$r /"
done
timeout 300 python tools/shape_sweep.py --rows 8 --alg online_fused --V 262144 16777216 --knob split_cta=0,2 --reps 7 2>&1 | grep -E "^\{" | sed "s/^/rows8 /"
