mkdir -p gpurun_out/grid
timeout 1500 python tools/grid_solve.py --out gpurun_out/grid/grid_cold.json > gpurun_out/grid/grid.log 2>&1
