set -x
timeout 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/g6_pytest.log 2>&1; tail -3 gpurun_out/g6_pytest.log
V="2048 3162 4096 5623 8192 10000 16384"
for gw in 2 4 8 16; do
python tools/shape_sweep.py --rows 4000 --alg online --V $V --set shape=4 --set staged_gw=$gw --knob staged_ng=1,2,3,4,6,8 --reps 5 > gpurun_out/g6_gw$gw.jsonl 2>&1
python tools/shape_sweep.py --rows 32768 --alg online --V 3162 5623 10000 --set shape=4 --set staged_gw=$gw --knob staged_ng=2,3,4,6 --reps 3 > gpurun_out/g6_many_gw$gw.jsonl 2>&1
done
python tools/shape_sweep.py --rows 4000 --alg online --V 2048 3162 4096 --knob shape=1,4 --reps 7 > gpurun_out/g6_res.jsonl 2>&1
