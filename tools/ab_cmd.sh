HFB_LIB=ab/libhfb_nobr.so timeout 100 python tools/debug_tma.py 70 45 58 | tr '\n' ' '; echo
for r in 1 2; do
  for L in ab/libhfb_now.so ab/libhfb_nobr.so; do
    echo -n "$L 512: "; HFB_LIB=$L timeout 120 python tools/time_step.py 512 512 58 2>&1 | tail -1
    echo -n "$L C4 full: "; HFB_LIB=$L timeout 120 python tools/time_step.py 1581 1301 58 full 2>&1 | tail -1
  done
done
