# step kernel: mid-column K loop unrolled x2 (ab/libhfb_unr2.so) now that the allocation
# has headroom (109 registers) vs the product (ab/libhfb_uw2.so)
HFB_LIB=ab/libhfb_unr2.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "north_star or full_size_dycore or c2_dycore_100 or rk3_step_c2" 2>&1 | tail -1
for r in 1 2 3; do
  for L in ab/libhfb_uw2.so ab/libhfb_unr2.so; do
    echo "== $L"
    HFB_LIB=$L timeout 300 python tools/time_step.py 1581 1301 58 full 2>&1 | tail -1
    HFB_LIB=$L timeout 300 python tools/time_step.py 1581 1301 58 dycore 2>&1 | tail -1
  done
done
