# ASUCA pass A ring depth 5 vs 4
timeout 300 python tools/debug_asuca.py 128 96 58 2>&1 | tail -2
HFB_LIB=ab/libhfb_a5.so timeout 300 python tools/debug_asuca.py 128 96 58 2>&1 | tail -2
for r in 1 2; do for L in ab/libhfb_a4.so ab/libhfb_a5.so; do
  echo "$L"; HFB_LIB=$L timeout 300 python tools/time_step.py 1581 1301 58 asuca 2>&1 | tail -5 | head -3
done; done
