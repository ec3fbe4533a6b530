mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ab/pytest_pdl.log 2>&1
python tools/ab_time.py tools/ab/libB_pdl.so,STROM_PDL=80 tools/ab/libB_pdl.so 30 3 > gpurun_out/ab/pdl_pend30.txt 2>&1
python tools/ab_time.py tools/ab/libB_pdl.so,STROM_PDL=80 tools/ab/libB_pdl.so cartpole30 2 > gpurun_out/ab/pdl_cartpole30.txt 2>&1
