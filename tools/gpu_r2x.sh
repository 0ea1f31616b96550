# C1 (128x128x58): the fused step vs the split (K-parallel advection + acoustic) and
# single-role variants
for v in product split single_role generic; do
  echo -n "$v: "; timeout 120 python tools/time_step.py 128 128 58 dycore exact 0 $v 2>&1 | tail -1
  echo -n "$v 256: "; timeout 120 python tools/time_step.py 256 256 58 dycore exact 0 $v 2>&1 | tail -1
done
