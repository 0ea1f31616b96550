# ASUCA tendency pass with x faces shared between lanes (ghost lane, 31-column tiles):
# parity of every ASUCA test, then interleaved C4 timings against the previous kernel
timeout 1200 python -m pytest tests -m gpu -x -q -k "asuca or sanitizer" 2>&1 | tail -3
for r in 1 2 3; do
  for L in ab/libhfb_base.so ab/libhfb_xshare.so; do
    echo "== $L"; HFB_LIB=$L timeout 300 python tools/time_step.py 1581 1301 58 asuca 2>&1 | tail -6
  done
done
