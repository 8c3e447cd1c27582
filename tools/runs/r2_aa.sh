# stream kernel CTA size per V (512 vs 1024 threads) for naive / safe / online
set -x
for V in 177828 316228 562341 1000000; do
for A in online safe naive; do
python tools/cell_ab.py --alg $A --rows 4000 --V $V --cfg shape=2,stream_threads=512 --cfg shape=2,stream_threads=1024 --rounds 2 --reps 3
done; done > gpurun_out/r2aa.txt 2>&1
python tools/cell_ab.py --alg online --rows 4000 --V 131072 --cfg shape=2,stream_threads=512 --cfg shape=2,stream_threads=1024 --cfg "" --rounds 2 --reps 5 >> gpurun_out/r2aa.txt 2>&1
python tools/cell_ab.py --alg online_unfused --rows 4000 --V 262144 --cfg "" --cfg stream_threads=1024 --rounds 2 --reps 3 >> gpurun_out/r2aa.txt 2>&1
cat gpurun_out/r2aa.txt
