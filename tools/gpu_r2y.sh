# occupancy sensitivity of the step kernel: 16 resident warps (2 CTAs/SM) vs 8 (1 CTA/SM)
for r in 1 2; do
for L in paper_1710_08616_b200/libhfb.so ab/libhfb_onecta.so; do
  echo -n "$L C4 full: "; HFB_LIB=$L timeout 120 python tools/time_step.py 1581 1301 58 full 2>&1 | tail -1
done
done
