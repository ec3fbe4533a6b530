python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "projection or 50_iter or full_size_pend or final_obj or extract" > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log; grep -n "Error" gpurun_out/pytest_gpu.log | head -5
python tools/ab_time.py .ab/r01 . 30 3 2>&1 | tail -2
