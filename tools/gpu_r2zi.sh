# TMA waiter: early non-blocking test of the level's barrier (early) vs wait at the end (cur2)
HFB_LIB=ab/libhfb_early.so timeout 300 python tools/debug_tma.py 300 200 58 2>&1 | tail -1
for r in 1 2 3; do
  for L in ab/libhfb_cur2.so ab/libhfb_early.so; do
    echo -n "$L "; HFB_LIB=$L timeout 120 python tools/time_sustained.py exact 2>&1 | tail -1
  done
done
