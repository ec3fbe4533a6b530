O=gpurun_out/refresh2
mkdir -p $O
for c in cartpole30 carback30 landing50 flying60 carback60 carback120 carback240; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --inner 20 --no-cpu-baseline --gap-seconds 0 --batch 0 > $O/bench_$c.json 2> $O/bench_$c.err
done
