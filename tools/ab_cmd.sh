for r in 1 2; do
  for L in ab/libhfb_base.so ab/libhfb_cur.so; do
    echo -n "$L 512: "; HFB_LIB=$L timeout 120 python tools/time_step.py 512 512 58 2>&1 | tail -1
  done
done
