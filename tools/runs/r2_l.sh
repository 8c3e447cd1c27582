# same-box A/B of 1-warp vs 4-warp CTAs; V-split C-ABI bench; measured DRAM bytes per sweep cell
set -x
for V in 16384 32768 65536; do python tools/cell_ab.py --alg online_fused --rows 4000 --V $V --cfg topk_block=32 --cfg topk_block=128 --rounds 3; done > gpurun_out/r2l_ab.txt 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --sweep off --cpu off --e2e off --vsplit on --detail-out gpurun_out/r2l_vsplit_detail.json > gpurun_out/r2l_vsplit.out 2> gpurun_out/r2l_vsplit.err
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/r2l_cells.csv python tools/dram_cells.py run --out gpurun_out/r2l_cells_plan.json > gpurun_out/r2l_cells.log 2>&1
cat gpurun_out/r2l_ab.txt; tail -c 1500 gpurun_out/r2l_vsplit.out; tail -3 gpurun_out/r2l_vsplit.err; tail -3 gpurun_out/r2l_cells.log
python tools/dram_cells.py merge gpurun_out/r2l_cells_plan.json gpurun_out/r2l_cells.csv gpurun_out/dram_cells_r02.json
