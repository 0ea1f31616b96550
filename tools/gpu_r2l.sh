HFB_LIB=ab/libhfb_tmadbg.so timeout 120 python tools/debug_tma.py 70 45 20 2>&1 | head -8
HFB_LIB=ab/libhfb_tma.so timeout 300 python tools/debug_tma.py 300 200 58 2>&1 | tail -5
HFB_LIB=ab/libhfb_tma.so timeout 300 compute-sanitizer --tool memcheck --print-limit 3 python tools/debug_tma.py 70 45 20 2>&1 | grep -v "Host Frame\|^=========         " | tail -6
HFB_LIB=ab/libhfb_tma.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "dycore or full or rk3 or north or variant" 2>&1 | tail -3
for r in 1 2; do
  for L in ab/libhfb_cpa.so ab/libhfb_tma.so; do
    echo -n "$L "; HFB_LIB=$L timeout 120 python tools/time_sustained.py exact 2>&1 | tail -1
    echo -n "$L C4 dycore: "; HFB_LIB=$L timeout 120 python tools/time_step.py 1581 1301 58 2>&1 | tail -1
    echo -n "$L 512 dycore: "; HFB_LIB=$L timeout 120 python tools/time_step.py 512 512 58 2>&1 | tail -1
  done
done
