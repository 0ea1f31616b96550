# TMA issue guarded by elect.sync instead of lane == 0 (ab/libhfb_el.so: no BRA.U.ANY loop
# left around any UTMALDG) vs lane == 0 (ab/libhfb_uw2.so): parity, interleaved timings
HFB_LIB=ab/libhfb_el.so timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
for r in 1 2 3; do
  for L in ab/libhfb_uw2.so ab/libhfb_el.so; do
    echo "== $L"
    HFB_LIB=$L timeout 300 python tools/time_step.py 1581 1301 58 full 2>&1 | tail -1
    HFB_LIB=$L timeout 300 python tools/time_step.py 1581 1301 58 dycore 2>&1 | tail -1
    HFB_LIB=$L timeout 300 python tools/time_step.py 128 128 58 dycore 2>&1 | tail -1
    HFB_LIB=$L timeout 300 python tools/time_step.py 1581 1301 58 asuca 2>&1 | tail -5 | grep -E "asuca_step"
  done
done
