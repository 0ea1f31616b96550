# quick timing: parity spot check + 512^2 and C4 step times (+ optional env A/B list)
timeout 100 python tools/debug_tma.py 512 512 58 | tr '\n' ' '; echo
timeout 100 python tools/debug_tma.py 70 45 58 | tr '\n' ' '; echo
for v in "" "$@"; do
  echo -n "[$v] "; env $v timeout 120 python tools/time_step.py 512 512 58 2>&1 | tail -1
done
timeout 120 python tools/time_step.py 1581 1301 58 2>&1 | tail -1
