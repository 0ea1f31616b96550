# three-role step kernel (12 warps, setmaxnreg 56/80/104; ws3) vs the two-role product
# (ws2r: the same file compiled without -dc) vs the product library
HFB_LIB=ab/libhfb_ws3.so timeout 300 python tools/debug_tma.py 300 200 58 2>&1 | tail -5
HFB_LIB=ab/libhfb_ws3.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "dycore or full or north" 2>&1 | tail -2
for r in 1 2; do
  for L in paper_1710_08616_b200/libhfb.so ab/libhfb_ws2r.so ab/libhfb_ws3.so; do
    echo -n "$L "; HFB_LIB=$L timeout 120 python tools/time_sustained.py exact 2>&1 | tail -1
    echo -n "$L C4 dycore: "; HFB_LIB=$L timeout 120 python tools/time_step.py 1581 1301 58 2>&1 | tail -1
  done
done
