# Interleaved A/B timings of several builds of libhfb.so at C4 (full step and dycore step)
# usage: bash tools/ab_many.sh REPS lib1.so lib2.so ...
R=$1; shift
for r in $(seq $R); do
  for L in "$@"; do
    echo -n "$L full: "; HFB_LIB=$L timeout 120 python tools/time_step.py 1581 1301 58 full 2>&1 | tail -1
    echo -n "$L dycore: "; HFB_LIB=$L timeout 120 python tools/time_step.py 1581 1301 58 2>&1 | tail -1
  done
done
