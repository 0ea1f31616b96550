# step kernel: the TMA ring cursor (slot offset, barrier, level) shuffled from lane 0 so the
# issue operands are provably uniform (ab/libhfb_uw2.so) vs the uniform warp index alone
# (ab/libhfb_uw.so): parity, interleaved timings
HFB_LIB=ab/libhfb_uw2.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tolerance.py -q -x 2>&1 | tail -1
for r in 1 2 3; do
  for L in ab/libhfb_uw.so ab/libhfb_uw2.so; do
    echo "== $L"
    HFB_LIB=$L timeout 300 python tools/time_step.py 1581 1301 58 full 2>&1 | tail -1
    HFB_LIB=$L timeout 300 python tools/time_step.py 1581 1301 58 dycore 2>&1 | tail -1
    HFB_LIB=$L timeout 300 python tools/time_step.py 512 512 58 rk3 2>&1 | tail -1
    HFB_LIB=$L timeout 300 python tools/time_step.py 128 128 58 dycore 2>&1 | tail -1
  done
done
