set -x
timeout 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/g5_pytest.log 2>&1; tail -3 gpurun_out/g5_pytest.log
V="562 1000 1023 1778 2048 3162 4096 5623 8192 10000 16384"
python tools/shape_sweep.py --rows 4000 --alg online --V $V --knob shape=1,4 --reps 7 > gpurun_out/g5_a.jsonl 2>&1
python tools/shape_sweep.py --rows 4000 --alg online --V $V --set shape=4 --knob staged_cfg=1,2,3 --reps 7 > gpurun_out/g5_b.jsonl 2>&1
python tools/shape_sweep.py --rows 32768 --alg online --V 1000 1778 3162 5623 10000 --set shape=4 --knob staged_cfg=1,2,3 --reps 5 > gpurun_out/g5_c.jsonl 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_softmax_staged -c 1 -o gpurun_out/g5_staged5623 python tools/run_op.py --alg online --rows 4000 --V 5623 --reps 1 > /dev/null 2>&1
