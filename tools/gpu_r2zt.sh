# acoustic passes: TMA boxes issued by the horizontal warps only in pass A (ab/libhfb_acoh.so) vs by
# all eight warps (ab/libhfb_base.so): ASUCA parity with the new build, interleaved C4 timings
HFB_LIB=ab/libhfb_acoh.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k asuca 2>&1 | tail -2
for r in 1 2 3; do
  for L in ab/libhfb_base.so ab/libhfb_acoh.so; do
    echo "== $L"; HFB_LIB=$L timeout 300 python tools/time_step.py 1581 1301 58 asuca 2>&1 | tail -5
  done
done
