# the final tree once more: full GPU suite, smoke, the bench line and the ASUCA line
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_v9.json 2> gpurun_out/bench_v9.err; tail -1 gpurun_out/bench_v9.err
cut -c1-400 gpurun_out/bench_v9.json
timeout 900 python bench.py --entry asuca_step --steps 10 --warmup 3 > gpurun_out/bench_asuca_v9.json 2> gpurun_out/bench_asuca_v9.err; tail -1 gpurun_out/bench_asuca_v9.err
cut -c1-300 gpurun_out/bench_asuca_v9.json
