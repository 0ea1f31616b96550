# TMA-fed step (fixed static smem alignment) vs cp.async feed; parity of both; ncu of the
# warp-specialised ASUCA acoustic passes
set -x
HFB_LIB=ab/libhfb_tma.so timeout 300 python tools/debug_tma.py 300 200 58 2>&1 | tail -5
HFB_LIB=ab/libhfb_tma.so timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python tools/debug_tma.py 70 45 20 2>&1 | tail -4
HFB_LIB=ab/libhfb_tma.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "dycore or full or rk3 or north or variant" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "dycore or full or rk3 or north or variant" 2>&1 | tail -3
set +x
for r in 1 2; do
  for L in ab/libhfb_cpa.so ab/libhfb_tma.so; do
    echo -n "$L "; HFB_LIB=$L timeout 120 python tools/time_sustained.py exact 2>&1 | tail -1
    echo -n "$L C4 dycore: "; HFB_LIB=$L timeout 120 python tools/time_step.py 1581 1301 58 2>&1 | tail -1
    echo -n "$L 512 dycore: "; HFB_LIB=$L timeout 120 python tools/time_step.py 512 512 58 2>&1 | tail -1
  done
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_asu_acoustic -c 2 -o gpurun_out/prof_asu_r2j python tools/profile_step.py --entry asuca_step --steps 1 > gpurun_out/ncu_asu_r2j.log 2>&1
tail -1 gpurun_out/ncu_asu_r2j.log
