python tools/quick_time.py 2>&1 | grep -E "us/iter"
STROM_XSKIP_EIG=1 python tools/quick_time.py 2>&1 | grep -E "us/iter"
STROM_XSKIP_SOLVE=1 python tools/quick_time.py 2>&1 | grep -E "us/iter"
STROM_XSKIP_SOLVE=1 STROM_XSKIP_EIG=1 python tools/quick_time.py 2>&1 | grep -E "us/iter"
