# same-box A/B: 4000 x 32K fused top-K variants; 562K / 316K online stream knobs; 177K cluster sizes
set -x
python tools/cell_ab.py --alg online_fused --rows 4000 --V 32768 --cfg "" --cfg topk_block=128 --cfg topk_pipe=6 --cfg topk_pipe=1 --cfg topk_threads=32,topk_u8=1 --cfg tma=2 --cfg l2_prefetch=2 --rounds 3 > gpurun_out/r2z_32k.txt 2>&1
python tools/cell_ab.py --alg online_fused --rows 4000 --V 16384 --cfg "" --cfg topk_block=128 --cfg topk_pipe=6 --cfg topk_threads=32,topk_u8=1 --cfg tma=2 --rounds 3 > gpurun_out/r2z_16k.txt 2>&1
python tools/cell_ab.py --alg online --rows 4000 --V 562341 --cfg "" --cfg stream_threads=1024 --cfg stream_threads=256 --cfg stream_ctas=1 --cfg stream_ctas=2 --rounds 2 --reps 5 > gpurun_out/r2z_562k.txt 2>&1
python tools/cell_ab.py --alg safe --rows 4000 --V 562341 --cfg "" --cfg shape=2 --rounds 2 --reps 5 >> gpurun_out/r2z_562k.txt 2>&1
python tools/cell_ab.py --alg online --rows 4000 --V 177828 --cfg "" --cfg cluster_size=9 --cfg cluster_size=12 --cfg cluster_size=8 --cfg shape=2 --rounds 2 --reps 5 > gpurun_out/r2z_177k.txt 2>&1
cat gpurun_out/r2z_*.txt
