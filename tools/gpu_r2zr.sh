# final tree: the full GPU round (tests, smoke, bench + reference arm, launch list, ncu of
# the step kernel), the ASUCA line and an ncu capture of the ASUCA passes
bash tools/gpu_round.sh v6 ref
timeout 900 python bench.py --entry asuca_step --steps 10 --warmup 3 > gpurun_out/bench_asuca_v6.json 2> gpurun_out/bench_asuca_v6.err; tail -2 gpurun_out/bench_asuca_v6.err
cut -c1-600 gpurun_out/bench_asuca_v6.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_asu -c 4 -o gpurun_out/prof_asu_v6 python tools/profile_step.py --entry asuca_step --steps 1 > gpurun_out/ncu_asu_v6.log 2>&1
tail -2 gpurun_out/ncu_asu_v6.log
