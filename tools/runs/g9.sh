set -x
python tools/shape_sweep.py --rows 4000 --alg online safe --V 17783 31623 100000 316228 1000000 --set stream_threads=1024 --set stream_ctas=1 --knob l2_prefetch=0,1,2,3 --reps 5 > gpurun_out/g9_a.jsonl 2>&1
python tools/shape_sweep.py --rows 4000 --alg online safe --V 17783 31623 100000 316228 1000000 --set stream_threads=512 --set stream_ctas=2 --knob l2_prefetch=0,1,2,4 --reps 5 > gpurun_out/g9_b.jsonl 2>&1
python tools/shape_sweep.py --rows 4000 --alg online safe --V 17783 31623 100000 316228 1000000 --knob l2_prefetch=0,1,2 --reps 5 > gpurun_out/g9_c.jsonl 2>&1
