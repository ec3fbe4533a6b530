for k in none eig1 sep gemv p6a p1 p7 "sep,gemv" "eig0"; do
  echo -n "skip=$k: "; STROM_XSKIP=$k QT_NOSOLVE=1 python tools/quick_time.py 2>&1 | grep -E "N=30: .*us/iter" | cut -c1-40
done
