timeout 300 python tools/shape_sweep.py --rows 4000 --alg online_fused --V 16384 32768 65536 --knob topk_pipe=0,1,2,3,4,5,6 --reps 9 2>&1 | grep -E "^\{"
timeout 300 python tools/shape_sweep.py --rows 4000 --alg online_fused --V 16384 32768 65536 --set topk_pipe=0 --knob topk_u8=0,1 --reps 9 2>&1 | grep -E "^\{" | sed "s/^/p0 /"
