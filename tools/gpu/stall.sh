mkdir -p gpurun_out/stall
timeout 1800 python tools/sigma_stall.py 10000 > gpurun_out/stall/sigma_stall.jsonl 2>&1
