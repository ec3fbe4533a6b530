mkdir -p gpurun_out/ttt
timeout 1500 python tools/time_to_tol_models.py --out gpurun_out/ttt/time_to_tol_models.json > gpurun_out/ttt/ttt.log 2>&1
