mkdir -p gpurun_out/ab
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ab/pytest_ch16.log 2>&1
STROM_GEMV_CHUNK=16 timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "solve_parity or 50_iter or full_size or batched" > gpurun_out/ab/pytest_ch16_forced.log 2>&1
for c in landing50 flying60 carback30 cartpole30; do
python tools/ab_time.py tools/ab/libB_ch16.so,STROM_GEMV_CHUNK=8 tools/ab/libB_ch16.so $c 2 > gpurun_out/ab/ch16_$c.txt 2>&1
done
python tools/ab_time.py tools/ab/libB_ch16.so tools/ab/libB_ch16.so,STROM_GEMV_CHUNK=16 30 2 > gpurun_out/ab/ch16_pend30.txt 2>&1
