O=gpurun_out/lists
mkdir -p $O
for c in carback30 landing50; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"^k_" -s 100 -c 100 --csv --log-file $O/launches_$c.csv python tools/prof_run.py $c 12 > /dev/null 2>&1
  python tools/launches_warm.py $O/launches_$c.csv 5 > $O/launches_summary_$c.txt 2>&1
done
