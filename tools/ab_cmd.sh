for r in 1 2; do
  for L in ab/libhfb_now.so ab/libhfb_extradevicevectoriza.so ab/libhfb_XptxasO2.so ab/libhfb_Xptxasallowexpensive.so; do
    echo -n "$L 512: "; HFB_LIB=$L timeout 120 python tools/time_step.py 512 512 58 2>&1 | tail -1
  done
done
