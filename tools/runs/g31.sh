./build/read_peak
python tools/shape_sweep.py --rows 65536 --alg online_fused --V 131072 --knob l2_prefetch=0,1,2,3 --reps 5
python tools/shape_sweep.py --rows 65536 --alg online_fused --V 131072 --set topk_threads=32 --knob topk_u8=0,1 --reps 5
