for r in 1 2; do
for v in "HFB_DEBUG_SKIP=0" "HFB_DEBUG_SKIP=16" "HFB_DEBUG_SKIP=3" "HFB_DEBUG_SKIP=19"; do
  echo -n "[$v] "; env $v timeout 120 python tools/time_step.py 512 512 58 2>&1 | tail -1
done
done
