# ASUCA tendencies warp-specialised (scalars + w / u, v) vs one role; waiter warp 7 or 3
timeout 300 compute-sanitizer --tool memcheck --print-limit 3 python tools/debug_asuca.py 128 96 58 2>&1 | grep -v "Host Frame\|^=========         " | tail -6
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hfc.py tests/test_gpu_peer.py -q -x -p no:cacheprovider -k "asuca" 2>&1 | tail -3
for r in 1 2; do
for L in ab/libhfb_asutma.so ab/libhfb_tendws7.so ab/libhfb_tendws3.so; do
  echo "$L asuca:"; HFB_LIB=$L timeout 300 python tools/time_step.py 1581 1301 58 asuca 2>&1 | tail -5 | head -2
done
done
