mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "kernel_work or pooled" > gpurun_out/ab/pytest_new.log 2>&1
