# replicate r2_ad's first command, bounded; then each kb in one process, bounded
set -x
timeout 240 python tools/cell_ab.py --alg online --rows 4000 --V 7500 --cfg "" --cfg staged_kb=120 --cfg staged_kb=140 --cfg staged_kb=160 --cfg staged_kb=180 --cfg staged_kb=200 --rounds 3 --reps 10 > gpurun_out/r2ag_a.txt 2>&1; echo "a rc=$?" >> gpurun_out/r2ag_status.txt
timeout 120 python tools/cell_ab.py --alg online --rows 4000 --V 7500 --cfg "" --cfg staged_kb=120 --rounds 1 --reps 3 > gpurun_out/r2ag_b.txt 2>&1; echo "b rc=$?" >> gpurun_out/r2ag_status.txt
timeout 120 python tools/cell_ab.py --alg online --rows 4000 --V 7500 --cfg staged_kb=180 --cfg staged_kb=200 --rounds 1 --reps 3 > gpurun_out/r2ag_c.txt 2>&1; echo "c rc=$?" >> gpurun_out/r2ag_status.txt
cat gpurun_out/r2ag_status.txt gpurun_out/r2ag_?.txt
