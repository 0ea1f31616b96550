# acoustic-only TMA issuers with the waiter on an acoustic warp (3 or 2) vs advection warp 4
HFB_LIB=ab/libhfb_acW3.so timeout 300 python tools/debug_tma.py 300 200 58 2>&1 | tail -1
for r in 1 2 3; do
  for L in ab/libhfb_acOnly.so ab/libhfb_acW3.so ab/libhfb_acW2.so; do
    echo -n "$L "; HFB_LIB=$L timeout 120 python tools/time_sustained.py exact 2>&1 | tail -1
  done
done
