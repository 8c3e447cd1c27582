python tools/shape_sweep.py --rows 4000 --alg online_fused --V 32768 131072 1048576 --knob topk_minb=4,5,6
python tools/shape_sweep.py --rows 65536 --alg online_fused --V 131072 --knob topk_minb=4,5,6 --reps 5
