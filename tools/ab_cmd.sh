HFB_LIB=ab/libhfb_stcs.so timeout 100 python tools/debug_tma.py 70 45 58 | tr '\n' ' '; echo
for r in 1 2; do
  for L in ab/libhfb_now.so ab/libhfb_stcs.so; do
    echo -n "$L 512: "; HFB_LIB=$L timeout 120 python tools/time_step.py 512 512 58 2>&1 | tail -1
    echo -n "$L C4: "; HFB_LIB=$L timeout 120 python tools/time_step.py 1581 1301 58 2>&1 | tail -1
  done
done
HFB_LIB=ab/libhfb_stcs.so ncu --metrics dram__bytes.sum -k regex:k_dyn_step_ws -s 3 -c 1 python tools/time_step.py 512 512 58 2>&1 | grep dram__bytes
