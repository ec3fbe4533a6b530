python tools/quick_time.py 2>&1 | grep -E "us/iter"
STROM_PDL=0 python tools/quick_time.py 2>&1 | grep -E "us/iter"
python tools/shapes_time.py cartpole:30 2>&1 | python -c "import sys,json; [print(json.loads(l)['shape'], round(json.loads(l)['ms_per_iter']*1000,1),'us') for l in sys.stdin if l.startswith('{')]"
STROM_PDL=0 python tools/shapes_time.py cartpole:30 2>&1 | python -c "import sys,json; [print(json.loads(l)['shape'], round(json.loads(l)['ms_per_iter']*1000,1),'us') for l in sys.stdin if l.startswith('{')]"
