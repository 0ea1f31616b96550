set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; free -g | head -2
bash tools/gpu_round.sh r2a ref > gpurun_out/round_r2a.log 2>&1
tail -40 gpurun_out/round_r2a.log
for r in 1 2; do
  for L in paper_1710_08616_b200/libhfb.so paper_1710_08616_b200/libhfb_variants.so; do
    echo -n "$L C4 full: "; HFB_LIB=$L timeout 120 python tools/time_step.py 1581 1301 58 full 2>&1 | tail -1
    echo -n "$L C4 dycore: "; HFB_LIB=$L timeout 120 python tools/time_step.py 1581 1301 58 2>&1 | tail -1
  done
done
