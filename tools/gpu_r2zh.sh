# column physics in the acoustic warps (physAc) vs in the advection warps (physAdv)
HFB_LIB=ab/libhfb_physAc.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer.py tests/test_gpu_tolerance.py -q -x -p no:cacheprovider -k "full or north" 2>&1 | tail -2
for r in 1 2 3; do
  for L in ab/libhfb_physAdv.so ab/libhfb_physAc.so; do
    echo -n "$L "; HFB_LIB=$L timeout 120 python tools/time_sustained.py exact 2>&1 | tail -1
  done
done
