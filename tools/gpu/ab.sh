mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ab/pytest_yc.log 2>&1
for c in 30 landing50 flying60; do
python tools/ab_time.py tools/ab/libA_head.so tools/ab/libB_yc.so $c 2 > gpurun_out/ab/yc3_$c.txt 2>&1
done
