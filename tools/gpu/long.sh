O=gpurun_out/long
mkdir -p $O
nvidia-smi --query-gpu=name,memory.total --format=csv > $O/smi.txt 2>&1
for c in carback30 carback60 carback120 carback240; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --inner 20 --no-cpu-baseline --gap-seconds 0 > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_eig_cl" -s 4 -c 1 -o $O/full_carback30_k_eig_cl python tools/prof_run.py carback30 4 > $O/ncu_cl.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" -s 100 -c 100 --csv --log-file $O/launches_carback30.csv python tools/prof_run.py carback30 12 > /dev/null 2>&1
