timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_decomp.py -q -x -k "diffusion" 2>&1 | tail -1
for r in 1 2 3; do
  for L in ab/libhfb_now.so ab/libhfb_diff2.so; do
    echo -n "$L C4 diff: "; HFB_LIB=$L timeout 120 python tools/time_step.py 1581 1301 58 diffusion 2>&1 | tail -1
  done
done
echo -n "512 diff: "; timeout 120 python tools/time_step.py 512 512 58 diffusion 2>&1 | tail -1
