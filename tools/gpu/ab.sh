mkdir -p gpurun_out/ab
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "solve_parity or 50_iter or full_size or batched" > gpurun_out/ab/pytest_rowmaj.log 2>&1
for c in landing50 flying60 carback30 cartpole30; do
python tools/ab_time.py tools/ab/libB_rowmaj.so,STROM_GEMV_CHUNK_MAJOR=1 tools/ab/libB_rowmaj.so $c 2 > gpurun_out/ab/rowmaj_$c.txt 2>&1
done
python tools/ab_time.py tools/ab/libB_rowmaj.so,STROM_GEMV_CHUNK_MAJOR=1 tools/ab/libB_rowmaj.so 30 3 > gpurun_out/ab/rowmaj_pend30.txt 2>&1
