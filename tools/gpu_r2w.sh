# TMA issue by the advection warps (adviss) / by warps 0-5 with compile-time roles (aciss)
# vs HEAD (warps 0-5, runtime roles)
HFB_LIB=ab/libhfb_adviss.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "dycore or full or rk3 or north" 2>&1 | tail -2
for r in 1 2; do
  for L in ab/libhfb_head.so ab/libhfb_adviss.so ab/libhfb_aciss.so; do
    echo -n "$L "; HFB_LIB=$L timeout 120 python tools/time_sustained.py exact 2>&1 | tail -1
    echo -n "$L C4 dycore: "; HFB_LIB=$L timeout 120 python tools/time_step.py 1581 1301 58 2>&1 | tail -1
    echo -n "$L rk3: "; HFB_LIB=$L timeout 120 python tools/time_step.py 512 512 58 rk3 2>&1 | tail -1
  done
done
