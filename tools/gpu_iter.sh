# quick iteration: dycore parity subset, A/B timing (TMA vs cp.async), optional ncu capture
TAG=${1:-i}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "dycore or rk3 or full or graph or cpasync or division or smoke" 2>&1 | tail -4
for v in "" "HFB_TMA_STEP=1"; do
  echo "== $v"; env $v timeout 120 python tools/time_step.py 512 512 58 2>&1 | tail -1
done
timeout 120 python tools/time_step.py 1581 1301 58 2>&1 | tail -1
if [ -n "$2" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dyn_step -s 1 -c 1 -o gpurun_out/prof_$TAG python tools/profile_step.py --steps 2 > gpurun_out/ncu_$TAG.log 2>&1
  tail -1 gpurun_out/ncu_$TAG.log
fi
