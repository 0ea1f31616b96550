# L2 prefetch distance sweep for the fused step (HFB_L2_PREFETCH levels beyond the ring)
timeout 100 python tools/debug_tma.py 512 512 58 | tr '\n' ' '; echo
for pf in 0 2 4 6 8 12; do
  echo -n "pf=$pf: "; HFB_L2_PREFETCH=$pf timeout 120 python tools/time_step.py 512 512 58 2>&1 | tail -1
  echo -n "pf=$pf skel: "; HFB_DEBUG_SKIP=3 HFB_L2_PREFETCH=$pf timeout 120 python tools/time_step.py 512 512 58 2>&1 | tail -1
done
HFB_L2_PREFETCH=4 timeout 120 python tools/time_step.py 1581 1301 58 2>&1 | tail -1
