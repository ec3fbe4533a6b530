#!/bin/bash
# Round-2 measurement pass on one B200 (run under gpurun from the repo root):
# bench lines, steady-state launch lists and one `ncu --set full` capture per kernel.
set -x
O=gpurun_out/r02
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python bench.py > $O/bench_pend30.json 2> $O/bench_pend30.err
# launch lists (serialised, cold-cache: compare shares): skip the first 10 iterations
for c in pend30 carback30; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" -s 220 -c 220 \
     --csv --log-file $O/launches_$c.csv python tools/prof_run.py $c 25 > /dev/null 2>&1
  python tools/launches.py $O/launches_$c.csv > $O/launches_summary_$c.txt 2>&1
done
# one full capture per kernel family (pend30), after 10 warm iterations
for k in k_eig k_gemv_stage k_sep_tri k_solve_p1 k_solve_p3 k_solve_p6a k_solve_p7 k_update k_spmv_ax; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^$k(\$|<)" -s 20 -c 2 \
     -o $O/full_pend30_$k python tools/prof_run.py pend30 14 > /dev/null 2>&1
done
# the cluster K-EIG (order 190, car back-in) and its stage GEMV
for k in k_eig_cluster k_gemv_stage; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 4 -c 1 \
     -o $O/full_carback30_$k python tools/prof_run.py carback30 4 > /dev/null 2>&1
done
ls -la $O
