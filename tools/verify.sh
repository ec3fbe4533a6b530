set -x
O=gpurun_out/v0
mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" -s 220 -c 220 --csv --log-file $O/launches_pend30.csv python tools/prof_run.py pend30 25 > /dev/null 2>&1
python tools/launches.py $O/launches_pend30.csv > $O/launches_summary_pend30.txt 2>&1
