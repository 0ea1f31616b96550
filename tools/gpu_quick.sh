# quick GPU iteration: dycore parity, bench line, ncu of the dycore kernels
set -x
mkdir -p gpurun_out
TAG=${1:-q}
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "dycore or graph or smoke or role or split or generic" 2>&1 | tail -5
timeout 400 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -3 gpurun_out/bench_$TAG.err
cat gpurun_out/bench_$TAG.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dyn -s 1 -c 2 -o gpurun_out/prof_$TAG python tools/profile_step.py --steps 3 > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_$TAG.log
