# whole-program (no -dc) product library: the full GPU suite and timings
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -4
for r in 1 2; do
  echo -n "C4 full sustained: "; timeout 120 python tools/time_sustained.py exact 2>&1 | tail -1
  echo -n "asuca: "; timeout 300 python tools/time_step.py 1581 1301 58 asuca 2>&1 | tail -5 | head -1
done
