python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
mkdir -p gpurun_out/sanitize
for t in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_run.py > gpurun_out/sanitize/$t.log 2>&1
  echo "$t rc=$?"; tail -3 gpurun_out/sanitize/$t.log
done
