python tools/ab/hist2.py 2>&1 | grep iter
QT_NOSOLVE=1 python tools/quick_time.py 2>&1 | grep -E "us/iter" | cut -c1-60
STROM_FIRST_ORDER=0 QT_NOSOLVE=1 python tools/quick_time.py 2>&1 | grep -E "us/iter" | cut -c1-60
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
