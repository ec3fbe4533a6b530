O=gpurun_out/bench2
mkdir -p $O
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
