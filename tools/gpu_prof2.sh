# ncu full captures of the product step and its TMA twin (same inputs)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dyn_step -s 1 -c 1 -o gpurun_out/prof_cp python tools/profile_step.py --steps 2 > /dev/null 2>&1
HFB_TMA_STEP=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dyn_step -s 1 -c 1 -o gpurun_out/prof_tma python tools/profile_step.py --steps 2 > /dev/null 2>&1
HFB_TMA_STEP=1 HFB_DEBUG_SKIP=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dyn_step -s 1 -c 1 -o gpurun_out/prof_tma_s1 python tools/profile_step.py --steps 2 > /dev/null 2>&1
HFB_DEBUG_SKIP=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dyn_step -s 1 -c 1 -o gpurun_out/prof_cp_s1 python tools/profile_step.py --steps 2 > /dev/null 2>&1
ls gpurun_out
