# A/B timing of dycore variants (env switches) on one GPU + an ncu capture of the step kernel
TAG=${1:-ab}
for v in "" "HFB_DEBUG_SKIP=1" "HFB_DEBUG_SKIP=2" "HFB_DEBUG_SKIP=3"; do
  echo "== $v"; env $v timeout 120 python tools/time_step.py 512 512 58 2>&1 | tail -1
done
timeout 300 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "dycore or graph or role or split or generic" 2>&1 | tail -2
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_dyn_step -s 1 -c 1 -o gpurun_out/prof_$TAG python tools/profile_step.py --steps 2 > /dev/null 2>&1
echo ncu done
