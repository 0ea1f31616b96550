# round-2 re-entry: the full GPU check (tests, smoke, bench + reference arm, launch list,
# ncu of the step kernel) plus an ncu capture of the ASUCA step's kernels
TAG=r2f
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
bash tools/gpu_round.sh $TAG ref > gpurun_out/round_$TAG.log 2>&1
tail -40 gpurun_out/round_$TAG.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_asu -c 4 -o gpurun_out/prof_asu_$TAG python tools/profile_step.py --entry asuca_step --steps 1 > gpurun_out/ncu_asu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_asu_$TAG.log
echo done
