# co-run default for online at 16-CTA-cluster rows: parity (fullsize incl. new test), graph capture, full suite
set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2bk_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2bk_pytest.log
python tools/cell_ab.py --alg online --rows 4000 --V 177828 --cfg "" --cfg corun=0 --rounds 2 --reps 5 > gpurun_out/r2bk_ab.txt 2>&1
tail -3 gpurun_out/r2bk_pytest.log; grep online gpurun_out/r2bk_ab.txt
