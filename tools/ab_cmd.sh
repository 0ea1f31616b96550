for r in 1 2 3; do
  echo -n "C4 dyc: "; timeout 120 python tools/time_step.py 1581 1301 58 2>&1 | tail -1
  echo -n "C4 full: "; timeout 120 python tools/time_step.py 1581 1301 58 full 2>&1 | tail -1
done
