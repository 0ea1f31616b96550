# small grids: the three-role kernel (12 warps/tile, one CTA per SM) vs the two-role one;
# parity of the three-role kernel on every step test (forced everywhere: "always")
HFB_LIB=ab/libhfb_always.so timeout 300 python tools/debug_tma.py 300 200 58 2>&1 | tail -2
HFB_LIB=ab/libhfb_always.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer.py -q -p no:cacheprovider -k "dycore or full or rk3 or north or tall" 2>&1 | tail -4
for r in 1 2; do
  for L in ab/libhfb_nows3.so ab/libhfb_small.so; do
    echo -n "$L C1: "; HFB_LIB=$L timeout 120 python tools/time_step.py 128 128 58 2>&1 | tail -1
    echo -n "$L 160x160: "; HFB_LIB=$L timeout 120 python tools/time_step.py 160 160 58 2>&1 | tail -1
  done
done
echo -n "always C4 full: "; HFB_LIB=ab/libhfb_always.so timeout 120 python tools/time_step.py 1581 1301 58 full 2>&1 | tail -1
