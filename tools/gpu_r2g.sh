# A/B: role-split K loops (split) vs the previous kernel (base); parity subset on the new build
for r in 1 2; do
  for L in ab/libhfb_base.so ab/libhfb_split.so; do
    for a in exact fma; do echo -n "$L "; HFB_LIB=$L timeout 120 python tools/time_sustained.py $a 2>&1 | tail -1; done
    echo -n "$L C4 dycore: "; HFB_LIB=$L timeout 120 python tools/time_step.py 1581 1301 58 2>&1 | tail -1
    echo -n "$L 512 dycore: "; HFB_LIB=$L timeout 120 python tools/time_step.py 512 512 58 2>&1 | tail -1
    echo -n "$L 512 rk3: "; HFB_LIB=$L timeout 120 python tools/time_step.py 512 512 58 rk3 2>&1 | tail -1
    echo -n "$L 128 dycore: "; HFB_LIB=$L timeout 120 python tools/time_step.py 128 128 58 2>&1 | tail -1
  done
done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tolerance.py tests/test_gpu_peer.py -q -x -p no:cacheprovider 2>&1 | tail -4
