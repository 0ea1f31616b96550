# bench line + ncu launch list + full captures of the dycore step and the diffusion kernel
TAG=${1:-b}
mkdir -p gpurun_out
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -3 gpurun_out/bench_$TAG.err
cat gpurun_out/bench_$TAG.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python tools/profile_step.py --steps 5 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_dyn_step -s 1 -c 1 -o gpurun_out/prof_$TAG python tools/profile_step.py --steps 2 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_diffusion -s 1 -c 1 -o gpurun_out/profdiff_$TAG python tools/profile_step.py --app diffusion --nx 1581 --ny 1301 --steps 2 > /dev/null 2>&1
echo done
