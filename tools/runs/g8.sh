set -x
for th in 512 1024; do
python tools/shape_sweep.py --rows 4000 --alg online safe --V 31623 100000 316228 --set stream_threads=$th --knob stream_ctas=0,1,2 --reps 5 > gpurun_out/g8_th$th.jsonl 2>&1
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_softmax -c 1 --csv --log-file gpurun_out/g8_keep100k.csv python tools/run_op.py --alg online --rows 4000 --V 100000 --reps 1 --set stream_ctas=1 --set stream_threads=1024 > /dev/null 2>&1
