mkdir -p gpurun_out/batch
python tools/batched.py 4 8 16 > gpurun_out/batch/default.jsonl 2>&1
STROM_EIG_THREADS=256 python tools/batched.py 4 8 16 > gpurun_out/batch/t256.jsonl 2>&1
