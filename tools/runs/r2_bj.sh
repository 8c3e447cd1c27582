# 177828: co-run the 16-CTA cluster kernel with the streaming kernel on a side stream
set -x
for A in online safe; do
python tools/cell_ab.py --alg $A --rows 4000 --V 177828 --cfg "" --cfg corun=70 --cfg corun=75 --cfg corun=80 --cfg corun=85 --rounds 2 --reps 5 >> gpurun_out/r2bj_ab.txt 2>&1
done
python tools/cell_ab.py --alg online --rows 4000 --V 196000 --cfg "" --cfg corun=75 --cfg corun=80 --rounds 2 --reps 5 >> gpurun_out/r2bj_ab.txt 2>&1
grep -E "^(online|safe)" gpurun_out/r2bj_ab.txt; grep -i error gpurun_out/r2bj_ab.txt | head -3
