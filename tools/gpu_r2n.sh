# product = TMA-fed step + ASUCA acoustic formation in the Thomas warps: the full GPU suite,
# smoke, ASUCA A/B, the bench line, the launch list and ncu captures
TAG=r2n
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -8
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for L in ab/libhfb_cpa.so ab/libhfb_asu2.so; do
  echo "$L asuca:"; HFB_LIB=$L timeout 300 python tools/time_step.py 1581 1301 58 asuca 2>&1 | tail -5
done
timeout 900 python bench.py --steps 100 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -3 gpurun_out/bench_$TAG.err
cut -c1-1500 gpurun_out/bench_$TAG.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python tools/profile_step.py --steps 5 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dyn_step -s 1 -c 1 -o gpurun_out/prof_$TAG python tools/profile_step.py --steps 2 > gpurun_out/ncu_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_asu -c 4 -o gpurun_out/prof_asu_$TAG python tools/profile_step.py --entry asuca_step --steps 1 > gpurun_out/ncu_asu_$TAG.log 2>&1
tail -1 gpurun_out/ncu_$TAG.log gpurun_out/ncu_asu_$TAG.log
