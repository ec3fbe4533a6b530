for k in none eig0 eig1 sep p3 gemv p6a p1 p7; do
  echo -n "dup=$k: "; STROM_XDUP=$k QT_NOSOLVE=1 python tools/quick_time.py 2>&1 | grep -E "N=30: .*us/iter" | cut -c1-40
done
