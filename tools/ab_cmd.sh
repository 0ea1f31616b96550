# scratch A/B script for gpurun (edited per experiment); see ab_libs.sh for the library A/B
for L in ab/libhfb_now.so; do
  echo -n "$L 512: "; HFB_LIB=$L timeout 120 python tools/time_step.py 512 512 58 2>&1 | tail -1
done
