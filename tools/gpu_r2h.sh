# A/B: split vs chunk3 / unroll2; role balance (variants build, debug_skip)
for r in 1 2; do
  for L in ab/libhfb_split.so ab/libhfb_chunk3.so ab/libhfb_unroll2.so; do
    echo -n "$L "; HFB_LIB=$L timeout 120 python tools/time_sustained.py exact 2>&1 | tail -1
    echo -n "$L C4 dycore: "; HFB_LIB=$L timeout 120 python tools/time_step.py 1581 1301 58 2>&1 | tail -1
    echo -n "$L C4 full: "; HFB_LIB=$L timeout 120 python tools/time_step.py 1581 1301 58 full 2>&1 | tail -1
  done
done
for sk in 0 1 2; do
  echo -n "variants skip=$sk C4 full: "; HFB_LIB=paper_1710_08616_b200/libhfb_variants.so timeout 120 python tools/time_step.py 1581 1301 58 full exact $sk 2>&1 | tail -1
  echo -n "variants skip=$sk C4 dycore: "; HFB_LIB=paper_1710_08616_b200/libhfb_variants.so timeout 120 python tools/time_step.py 1581 1301 58 dycore exact $sk 2>&1 | tail -1
done
