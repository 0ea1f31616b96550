# acoustic pass B: TMA boxes issued by the Thomas warps (ab/libhfb_acob2.so) vs by every
# warp (ab/libhfb_acoh.so; both issue pass A's from the horizontal warps)
HFB_LIB=ab/libhfb_acob2.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "asuca_77 or asuca_128 or asuca_33x21" 2>&1 | tail -1
for r in 1 2 3; do
  for L in ab/libhfb_acoh.so ab/libhfb_acob2.so; do
    echo "== $L"; HFB_LIB=$L timeout 300 python tools/time_step.py 1581 1301 58 asuca 2>&1 | tail -5 | grep -E "asuca_step|acoustic"
  done
done
