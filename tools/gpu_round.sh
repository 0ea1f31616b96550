# full GPU check of the current tree: all gpu tests, smoke, bench line (+ the reference
# arm), the launch list and one ncu --set full capture of the dominant kernel at the
# headline workload (full_step, 1581x1301x58)
TAG=${1:-r}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -8
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py --steps 100 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -3 gpurun_out/bench_$TAG.err
cat gpurun_out/bench_$TAG.json
if [ -n "$2" ]; then
  timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; tail -3 gpurun_out/bench_ref_$TAG.err
  cat gpurun_out/bench_ref_$TAG.json
fi
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python tools/profile_step.py --steps 5 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dyn_step -s 1 -c 1 -o gpurun_out/prof_$TAG python tools/profile_step.py --steps 2 > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_$TAG.log
echo done
