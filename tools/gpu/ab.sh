mkdir -p gpurun_out/ab
L=paper_2406_05846_b200/libstrom.so
python tools/ab_time.py $L $L,STROM_GEMV_CTA_ROWS=1024 $L,STROM_GEMV_CTA_ROWS=512 30 3 > gpurun_out/ab/ctarows_pend30.txt 2>&1
