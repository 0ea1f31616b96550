# timing of dycore variants + quick parity
for v in "" "HFB_DEBUG_SKIP=1" "HFB_DEBUG_SKIP=2" "HFB_DEBUG_SKIP=3"; do
  echo "== $v"; env $v timeout 120 python tools/time_step.py 512 512 58 2>&1 | tail -1
done
timeout 120 python tools/time_step.py 1581 1301 58 2>&1 | tail -1
timeout 300 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "dycore or graph or role or split or generic or full or rk3" 2>&1 | tail -2
