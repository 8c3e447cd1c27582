# final: DRAM cells refresh (co-run at 177828), default bench, reference arm
set -x
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/r2bl_cells.csv python tools/dram_cells.py run --out gpurun_out/r2bl_cells_plan.json > gpurun_out/r2bl_cells.log 2>&1; echo "cells rc=$?" >> gpurun_out/r2bl_status.txt
python tools/dram_cells.py merge gpurun_out/r2bl_cells_plan.json gpurun_out/r2bl_cells.csv profiles/dram_cells_r02.json >> gpurun_out/r2bl_cells.log 2>&1; echo "merge rc=$?" >> gpurun_out/r2bl_status.txt
cp profiles/dram_cells_r02.json gpurun_out/r2bl_dram_cells_r02.json
timeout 900 python bench.py --detail-out gpurun_out/r2bl_detail.json > gpurun_out/r2bl_bench.out 2> gpurun_out/r2bl_bench.err; echo "bench rc=$?" >> gpurun_out/r2bl_status.txt
timeout 900 python bench.py --impl reference > gpurun_out/r2bl_ref.out 2> gpurun_out/r2bl_ref.err; echo "ref rc=$?" >> gpurun_out/r2bl_status.txt
cat gpurun_out/r2bl_status.txt; tail -c 1200 gpurun_out/r2bl_bench.out; tail -c 300 gpurun_out/r2bl_ref.out
