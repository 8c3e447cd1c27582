# synccheck after the non-aligned barrier in topk_large; large-k parity + timing
set -x
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_run.py > gpurun_out/r2bd_synccheck.txt 2>&1; echo "synccheck rc=$?" >> gpurun_out/r2bd_status.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "large" > gpurun_out/r2bd_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2bd_status.txt
for k in 100 1000; do python tools/cell_ab.py --alg online_fused --rows 4000 --V 131072 --k $k --cfg "" --rounds 2 --reps 5 >> gpurun_out/r2bd_ab.txt 2>&1; done
cat gpurun_out/r2bd_status.txt; tail -n 2 gpurun_out/r2bd_synccheck.txt; grep -E "at .*\+0x" gpurun_out/r2bd_synccheck.txt | sort | uniq -c | head -5; grep online gpurun_out/r2bd_ab.txt
