# A/B: TMA step vs cp.async step, with the HFB_DEBUG_SKIP role experiments
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 100 python tools/debug_tma.py 512 512 58 | tr '\n' ' '; echo
for base in "" "HFB_TMA_STEP=1"; do
  for sk in 0 1 2 3; do
    echo -n "$base skip=$sk: "; env $base HFB_DEBUG_SKIP=$sk timeout 120 python tools/time_step.py 512 512 58 2>&1 | tail -1
  done
done
