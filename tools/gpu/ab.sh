mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "projection or full_size or wide" > gpurun_out/ab/pytest_cl4.log 2>&1
for c in carback30 landing50 flying60; do
python tools/ab_time.py tools/ab/libA_head.so tools/ab/libB_cl4.so $c 2 > gpurun_out/ab/cl4_$c.txt 2>&1
done
