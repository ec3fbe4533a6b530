for c in carback:30 flying:60; do
python tools/shapes_time.py $c 2>&1 | python -c "import sys,json; [print(json.loads(l)['shape'], round(json.loads(l)['ms_per_iter'],3),'ms', json.loads(l)['top_kernels_ms']) for l in sys.stdin if l.startswith('{')]"
STROM_GEMV_CTA_ROWS=0 python tools/shapes_time.py $c 2>&1 | python -c "import sys,json; [print('warp-only', json.loads(l)['shape'], round(json.loads(l)['ms_per_iter'],3),'ms', json.loads(l)['top_kernels_ms']) for l in sys.stdin if l.startswith('{')]"
done
