mkdir -p gpurun_out/ab
STROM_FACTOR_STREAM=1 timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "solve_parity or 50_iter or final_obj or full_size" > gpurun_out/ab/pytest_chain_forced.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ab/pytest_chain.log 2>&1
for c in landing50 flying60 carback30; do
python tools/ab_time.py tools/ab/libB_chain.so,STROM_SEP_CHAIN=0 tools/ab/libB_chain.so $c 2 > gpurun_out/ab/chain_$c.txt 2>&1
done
python tools/ab_time.py tools/ab/libB_chain.so tools/ab/libB_chain.so,STROM_FACTOR_STREAM=1 30 2 > gpurun_out/ab/chain_pend30_forced.txt 2>&1
