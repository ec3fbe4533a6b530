mkdir -p gpurun_out/ab
STROM_SEP_YC=4 STROM_FACTOR_STREAM=1 STROM_BATCH_COMPACT=1 timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ab/pytest_forced_paths.log 2>&1
STROM_P3_DEDUP=0 timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "solve_parity or 50_iter or partition" > gpurun_out/ab/pytest_nodedup.log 2>&1
