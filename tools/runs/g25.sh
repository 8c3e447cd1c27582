set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "softmax" > gpurun_out/g25_pytest.log 2>&1; tail -2 gpurun_out/g25_pytest.log
python tools/c5_sweep.py split_chunk=0 split_chunk=0
python tools/shape_sweep.py --rows 4000 --alg online naive safe --V 177828 316228 1000000 --knob shape=2 --reps 5
