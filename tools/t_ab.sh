mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/ab/pytest_sep2.log 2>&1
python tools/ab_time.py tools/ab/libA_base.so tools/ab/libB_sep2.so landing50 2 > gpurun_out/ab/ab_sep2_landing50.txt 2>&1
python tools/ab_time.py tools/ab/libA_base.so tools/ab/libB_sep2.so carback30 2 > gpurun_out/ab/ab_sep2_carback30.txt 2>&1
python tools/ab_time.py tools/ab/libA_base.so tools/ab/libB_sep2.so 30 3 > gpurun_out/ab/ab_sep2_pend30.txt 2>&1
