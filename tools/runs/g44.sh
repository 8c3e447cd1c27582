timeout 300 python tools/c5_sweep.py split_cta=-1 2>&1 | tail -1
for r in 2 8 32 64; do
  timeout 300 python tools/shape_sweep.py --rows $r --alg online_fused --V 1048576 4194304 --knob split_cta=0,2 --reps 9 2>&1 | grep -E "^\{" | sed "s/^/rows$r /"
done
