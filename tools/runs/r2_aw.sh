# refresh measured DRAM bytes per sweep cell (current kernels); then full GPU suite; then default bench
set -x
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/r2aw_cells.csv python tools/dram_cells.py run --out gpurun_out/r2aw_cells_plan.json > gpurun_out/r2aw_cells.log 2>&1; echo "cells rc=$?" >> gpurun_out/r2aw_status.txt
python tools/dram_cells.py merge gpurun_out/r2aw_cells_plan.json gpurun_out/r2aw_cells.csv profiles/dram_cells_r02.json >> gpurun_out/r2aw_cells.log 2>&1; echo "merge rc=$?" >> gpurun_out/r2aw_status.txt
cp profiles/dram_cells_r02.json gpurun_out/r2aw_dram_cells_r02.json
timeout 2000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2aw_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2aw_status.txt
timeout 900 python bench.py --detail-out gpurun_out/r2aw_detail.json > gpurun_out/r2aw_bench.out 2> gpurun_out/r2aw_bench.err; echo "bench rc=$?" >> gpurun_out/r2aw_status.txt
cat gpurun_out/r2aw_status.txt; tail -3 gpurun_out/r2aw_pytest.log; tail -c 1200 gpurun_out/r2aw_bench.out; tail -3 gpurun_out/r2aw_cells.log
