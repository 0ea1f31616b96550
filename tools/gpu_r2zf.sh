# TMA issue by the acoustic warps only (0: th+u, 1: v+w, 2: p, 3: rho) vs warps 0-5
HFB_LIB=ab/libhfb_acOnly.so timeout 300 python tools/debug_tma.py 300 200 58 2>&1 | tail -2
for r in 1 2 3; do
  for L in ab/libhfb_cur.so ab/libhfb_acOnly.so; do
    echo -n "$L "; HFB_LIB=$L timeout 120 python tools/time_sustained.py exact 2>&1 | tail -1
  done
done
