mkdir -p gpurun_out/gemv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemv_stage" -s 4 -c 2 -o gpurun_out/gemv/full_landing_gemv python tools/prof_run.py landing50 3 > gpurun_out/gemv/ncu.log 2>&1
