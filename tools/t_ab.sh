mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ab/pytest_compact.log 2>&1
