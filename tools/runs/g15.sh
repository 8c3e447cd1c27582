set -x
python tools/shape_sweep.py --rows 4000 --alg online_fused --V 32768 65536 --set topk_u8=1 --set topk_threads=32 --knob l2_prefetch=0,1,2,4 --reps 7 > gpurun_out/g15_a.jsonl 2>&1
python tools/shape_sweep.py --rows 4000 --alg online_fused --V 32768 65536 --knob topk_threads=32,128,256,512 --reps 7 > gpurun_out/g15_b.jsonl 2>&1
python tools/shape_sweep.py --rows 4000 --alg online_fused --V 32768 65536 --knob tma=0,2 --reps 7 > gpurun_out/g15_c.jsonl 2>&1
python tools/shape_sweep.py --rows 4000 --alg online_fused --V 32768 65536 --knob shape=3 --set split_chunk=16384 --reps 7 > gpurun_out/g15_d.jsonl 2>&1
