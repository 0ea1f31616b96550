timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "full" 2>&1 | tail -1
timeout 300 python -m pytest tests/test_gpu_decomp.py -q -x -k "full" 2>&1 | tail -1
for r in 1 2; do
  for L in ab/libhfb_now.so ab/libhfb_physbal.so; do
    echo -n "$L 512 full: "; HFB_LIB=$L timeout 120 python tools/time_step.py 512 512 58 full 2>&1 | tail -1
    echo -n "$L C4 full: "; HFB_LIB=$L timeout 120 python tools/time_step.py 1581 1301 58 full 2>&1 | tail -1
  done
done
