mkdir -p gpurun_out/warm
timeout 1800 python tools/warm_grid.py --N 30 --db-theta 6 --db-dot 11 --every 7 --balance --carry-sigma --maxiter 5000 --out gpurun_out/warm/warm_grid.json > gpurun_out/warm/warm.log 2>&1
