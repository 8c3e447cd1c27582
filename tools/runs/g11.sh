set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "cluster or misaligned or nonfinite" > gpurun_out/g11_pytest.log 2>&1; tail -3 gpurun_out/g11_pytest.log
python tools/shape_sweep.py --rows 4000 --alg online --V 31623 100000 --set shape=5 --knob cluster_size=2,4,8,16 --reps 5 > gpurun_out/g11_b.jsonl 2>&1
python tools/shape_sweep.py --rows 4000 --alg online safe --V 17783 31623 56234 100000 177828 316228 --knob shape=2,5 --reps 5 > gpurun_out/g11_a.jsonl 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_softmax_cluster -c 1 -o gpurun_out/g11_cl100k python tools/run_op.py --alg online --rows 4000 --V 100000 --reps 1 --set shape=5 > /dev/null 2>&1
