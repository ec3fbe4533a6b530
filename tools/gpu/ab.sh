mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ab/pytest_p3d.log 2>&1
