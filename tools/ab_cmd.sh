for v in "HFB_DEBUG_SKIP=0" "HFB_DEBUG_SKIP=1" "HFB_DEBUG_SKIP=2" "HFB_DEBUG_SKIP=3"; do
  echo -n "[$v] dyc "; env $v timeout 120 python tools/time_step.py 512 512 58 2>&1 | tail -1
  echo -n "[$v] full "; env $v timeout 120 python tools/time_step.py 512 512 58 full 2>&1 | tail -1
done
