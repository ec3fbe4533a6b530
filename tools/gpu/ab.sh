mkdir -p gpurun_out/ab
L=paper_2406_05846_b200/libstrom.so
python tools/ab_time.py $L,STROM_P3_DEDUP=0 $L 30 5 > gpurun_out/ab/p3d_pend30_5.txt 2>&1
