O=gpurun_out/refresh
mkdir -p $O
for c in cartpole30 landing50 flying60; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --inner 20 --no-cpu-baseline --gap-seconds 0 --batch 0 > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 1500 python tools/grid_solve.py --out $O/grid_cold.json > $O/grid.log 2>&1
