# A/B two builds of libhfb.so: interleaved repeated timings (median reported by the caller)
# usage: bash tools/ab_libs.sh libA.so libB.so [reps]
A=$1; B=$2; R=${3:-3}
for r in $(seq $R); do
  for L in $A $B; do
    echo -n "$L 512: "; HFB_LIB=$L timeout 120 python tools/time_step.py 512 512 58 2>&1 | tail -1
    echo -n "$L C4: "; HFB_LIB=$L timeout 120 python tools/time_step.py 1581 1301 58 2>&1 | tail -1
  done
done
