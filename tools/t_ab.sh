mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/ab/pytest_dmma.log 2>&1
for v in 1 0; do STROM_EIG_DMMA=$v timeout 300 python tools/eig_prof.py 30 400 > gpurun_out/ab/prof_dmma$v.log 2>&1; done
python tools/ab_time.py tools/ab/libB_dmma.so,STROM_EIG_DMMA=0 tools/ab/libB_dmma.so 30 3 > gpurun_out/ab/ab_dmma_pend30.txt 2>&1
