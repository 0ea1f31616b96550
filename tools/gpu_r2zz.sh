# acoustic pass B issue policy re-measured with the warp-uniform index: every warp
# (ab/libhfb_uw2.so, the product), horizontal warps (ab/libhfb_bh.so), Thomas warps
# (ab/libhfb_bt.so)
for L in ab/libhfb_bh.so ab/libhfb_bt.so; do
  HFB_LIB=$L timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "asuca_77 or asuca_128 or asuca_93" 2>&1 | tail -1
done
for r in 1 2 3; do
  for L in ab/libhfb_uw2.so ab/libhfb_bh.so ab/libhfb_bt.so; do
    echo "== $L"; HFB_LIB=$L timeout 300 python tools/time_step.py 1581 1301 58 asuca 2>&1 | tail -5 | grep -E "asuca_step|acoustic_b"
  done
done
