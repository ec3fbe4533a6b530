mkdir -p gpurun_out/ab
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "projection or 50_iter or final_obj or full_size_pend" > gpurun_out/ab/pytest_uni.log 2>&1
python tools/ab_time.py tools/ab/libA_head.so tools/ab/libB_uni.so 30 4 > gpurun_out/ab/uni_pend30.txt 2>&1
python tools/ab_time.py tools/ab/libA_head.so tools/ab/libB_uni.so cartpole30 2 > gpurun_out/ab/uni_cartpole30.txt 2>&1
