# TMA L2 promotion of the plane boxes: 256 B (product) / 128 B / none
for r in 1 2; do
  for L in ab/libhfb_p256.so ab/libhfb_p128.so ab/libhfb_p0.so; do
    echo -n "$L "; HFB_LIB=$L timeout 120 python tools/time_sustained.py exact 2>&1 | tail -1
    echo -n "$L C4 dycore: "; HFB_LIB=$L timeout 120 python tools/time_step.py 1581 1301 58 2>&1 | tail -1
    echo -n "$L asuca: "; HFB_LIB=$L timeout 300 python tools/time_step.py 1581 1301 58 asuca 2>&1 | tail -5 | head -1
  done
done
