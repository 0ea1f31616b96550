set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
free -g | head -2; nproc
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 900 python -m pytest tests -m gpu -q --maxfail=30 -p no:cacheprovider 2>&1 | tail -40
timeout 400 python bench.py --steps 50 --warmup 5 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; tail -3 gpurun_out/bench1.err
cat gpurun_out/bench1.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches1.csv python tools/profile_step.py --steps 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dyn -s 2 -c 2 -o gpurun_out/prof_dycore1 python tools/profile_step.py --steps 3 > gpurun_out/ncu1.log 2>&1
tail -3 gpurun_out/ncu1.log
