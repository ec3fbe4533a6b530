mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/ab/pytest_blk.log 2>&1
for v in 1 0; do STROM_EIG_BLK=$v timeout 300 python tools/eig_prof.py 30 400 > gpurun_out/ab/prof_blk$v.log 2>&1; done
python tools/ab_time.py tools/ab/libB_blk.so,STROM_EIG_BLK=0 tools/ab/libB_blk.so 30 3 > gpurun_out/ab/blk_pend30.txt 2>&1
