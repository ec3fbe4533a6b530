mkdir -p gpurun_out/setup
STROM_PROF_SETUP=1 python tools/setup_time.py 30 8 > gpurun_out/setup/st2.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/setup/pytest.log 2>&1
