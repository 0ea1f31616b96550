# RK stages: L2 prefetch of the base state (TMA prefetch boxes) vs none
HFB_LIB=ab/libhfb_rkpf.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "rk3" 2>&1 | tail -2
for r in 1 2 3; do
for L in ab/libhfb_rk0.so ab/libhfb_rkpf.so; do
  echo -n "$L "; HFB_LIB=$L timeout 300 python tools/time_step.py 512 512 58 rk3 2>&1 | tail -1
  echo -n "$L "; HFB_LIB=$L timeout 300 python tools/time_step.py 1581 1301 58 rk3 2>&1 | tail -1
done
done
