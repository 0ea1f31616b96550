# C1 (128x128x58 dycore step): one ncu --set full capture, to show what bounds the small grid
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dyn_step -s 2 -c 1 -o gpurun_out/prof_c1 python tools/profile_step.py --entry dycore_step --nx 128 --ny 128 --steps 4 > gpurun_out/ncu_c1.log 2>&1
tail -2 gpurun_out/ncu_c1.log
