set -x
python tools/shape_sweep.py --rows 4000 --alg online --V 56234 100000 177828 --set shape=5 --knob cluster_size=3,4,5,6,7,8,9,12 --reps 5 > gpurun_out/g13_a.jsonl 2>&1
python tools/shape_sweep.py --rows 4000 --alg online --V 56234 100000 177828 --set shape=5 --set staged_gw=8 --knob cluster_size=4,6,8 --reps 5 > gpurun_out/g13_b.jsonl 2>&1
python tools/shape_sweep.py --rows 32768 --alg online --V 17783 31623 56234 --knob shape=2,5 --reps 3 > gpurun_out/g13_c.jsonl 2>&1
