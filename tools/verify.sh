# Round verification on one B200: smoke, GPU suite, bench line, steady-state launch list,
# one full ncu capture of the top kernel (run from the repo root under gpurun).
O=gpurun_out/${VERIFY_DIR:-final}
mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" -s 220 -c 220 --csv --log-file $O/launches_pend30.csv python tools/prof_run.py pend30 25 > /dev/null 2>&1
python tools/launches.py $O/launches_pend30.csv > $O/launches_summary_pend30.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_eig<.int.8" -s 10 -c 1 -o $O/full_pend30_k_eig python tools/prof_run.py pend30 14 > $O/ncu_full.log 2>&1
python tools/ncu_lines.py $O/full_pend30_k_eig.ncu-rep 0.01 > $O/ncu_lines_k_eig.txt 2>&1
