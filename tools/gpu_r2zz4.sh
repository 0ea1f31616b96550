# ncu of the final tree's step kernel (full_step C4) and launch list
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v9.csv python tools/profile_step.py --steps 5 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dyn_step -s 1 -c 1 -o gpurun_out/prof_v9 python tools/profile_step.py --steps 2 > gpurun_out/ncu_v9.log 2>&1
tail -1 gpurun_out/ncu_v9.log
