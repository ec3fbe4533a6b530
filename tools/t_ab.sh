mkdir -p gpurun_out/ab gpurun_out/final
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_eig<.int.8" -s 10 -c 1 -o gpurun_out/final/full_pend30_k_eig python tools/prof_run.py pend30 14 > gpurun_out/final/ncu_full.log 2>&1
python tools/ncu_lines.py gpurun_out/final/full_pend30_k_eig.ncu-rep 0.01 > gpurun_out/final/ncu_lines_k_eig.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/ab/pytest_cs.log 2>&1
python tools/ab_time.py tools/ab/libB_cs.so,STROM_FACTOR_STREAM=0 tools/ab/libB_cs.so landing50 2 > gpurun_out/ab/ab_cs_landing50.txt 2>&1
python tools/ab_time.py tools/ab/libB_cs.so,STROM_FACTOR_STREAM=0 tools/ab/libB_cs.so carback30 2 > gpurun_out/ab/ab_cs_carback30.txt 2>&1
python tools/ab_time.py tools/ab/libB_cs.so,STROM_FACTOR_STREAM=0 tools/ab/libB_cs.so flying60 2 > gpurun_out/ab/ab_cs_flying60.txt 2>&1
python tools/ab_time.py tools/ab/libB_cs.so tools/ab/libB_cs.so,STROM_FACTOR_STREAM=1 30 2 > gpurun_out/ab/ab_cs_pend30.txt 2>&1
