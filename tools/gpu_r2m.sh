# TMA feed: which warp waits on the slot barriers
HFB_LIB=ab/libhfb_tma0.so timeout 300 python tools/debug_tma.py 300 200 58 2>&1 | tail -5
for r in 1 2; do
  for L in ab/libhfb_tma4.so ab/libhfb_tma7.so ab/libhfb_tma0.so ab/libhfb_tma3.so; do
    echo -n "$L "; HFB_LIB=$L timeout 120 python tools/time_sustained.py exact 2>&1 | tail -1
    echo -n "$L C4 dycore: "; HFB_LIB=$L timeout 120 python tools/time_step.py 1581 1301 58 2>&1 | tail -1
    echo -n "$L C4 full: "; HFB_LIB=$L timeout 120 python tools/time_step.py 1581 1301 58 full 2>&1 | tail -1
  done
done
