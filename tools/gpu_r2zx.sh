# final tree (uniform warp index + cursor): the full GPU round, the ASUCA line, ncu of the
# step kernel and the ASUCA passes
bash tools/gpu_round.sh v7
timeout 900 python bench.py --entry asuca_step --steps 10 --warmup 3 > gpurun_out/bench_asuca_v7.json 2> gpurun_out/bench_asuca_v7.err; tail -2 gpurun_out/bench_asuca_v7.err
cut -c1-300 gpurun_out/bench_asuca_v7.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_asu -c 4 -o gpurun_out/prof_asu_v7 python tools/profile_step.py --entry asuca_step --steps 1 > gpurun_out/ncu_asu_v7.log 2>&1
tail -1 gpurun_out/ncu_asu_v7.log
