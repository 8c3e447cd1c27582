set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "staged or misaligned or nonfinite" > gpurun_out/g4_pytest.log 2>&1; tail -3 gpurun_out/g4_pytest.log
V="1000 1778 3162 5623 10000 16384"
python tools/shape_sweep.py --rows 4000 --alg online safe --V $V --knob shape=0,4 --reps 7 > gpurun_out/g4_c0.jsonl 2>&1
python tools/shape_sweep.py --rows 4000 --alg online safe --V $V --set shape=4 --knob staged_cfg=1 --reps 7 > gpurun_out/g4_c1.jsonl 2>&1
python tools/shape_sweep.py --rows 4000 --alg online safe --V $V --set shape=4 --set staged_kb=100 --knob staged_cfg=0,2 --reps 7 > gpurun_out/g4_c2.jsonl 2>&1
python tools/shape_sweep.py --rows 32768 --alg online --V 1000 3162 10000 --knob shape=0,4 --reps 5 > gpurun_out/g4_many.jsonl 2>&1
python tools/shape_sweep.py --rows 32768 --alg online --V 1000 3162 10000 --set shape=4 --set staged_kb=100 --knob staged_cfg=0,2 --reps 5 >> gpurun_out/g4_many.jsonl 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_softmax_staged -c 1 -o gpurun_out/g4_staged5623 python tools/run_op.py --alg online --rows 4000 --V 5623 --reps 1 --set shape=4 > /dev/null 2>&1
