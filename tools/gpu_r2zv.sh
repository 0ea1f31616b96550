# warp index shuffled from lane 0 (known warp-uniform: TMA issue without the per-lane
# waterfall, uniform role branches; ab/libhfb_uw.so) vs threadIdx.y (ab/libhfb_base.so):
# parity of the step / RK3 / ASUCA kernels with the new build, interleaved timings
HFB_LIB=ab/libhfb_uw.so timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
for r in 1 2; do
  for L in ab/libhfb_base.so ab/libhfb_uw.so; do
    echo "== $L"
    HFB_LIB=$L timeout 300 python tools/time_step.py 1581 1301 58 full 2>&1 | tail -1
    HFB_LIB=$L timeout 300 python tools/time_step.py 1581 1301 58 dycore 2>&1 | tail -1
    HFB_LIB=$L timeout 300 python tools/time_step.py 512 512 58 rk3 2>&1 | tail -1
    HFB_LIB=$L timeout 300 python tools/time_step.py 128 128 58 dycore 2>&1 | tail -1
    HFB_LIB=$L timeout 300 python tools/time_step.py 1581 1301 58 asuca 2>&1 | tail -5
  done
done
