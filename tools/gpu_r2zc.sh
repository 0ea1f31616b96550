# final round-2 measurement of the tree: smoke, the bench line and the reference arm, the
# multi-rank bench path on one GPU, launch list, ncu of the step and the ASUCA passes
TAG=r2zc
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 100 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -2 gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; tail -2 gpurun_out/bench_ref_$TAG.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 4 --steps 20 --warmup 3 --tile512 --one-gpu-test --no-secondary > gpurun_out/bench4_$TAG.json 2> gpurun_out/bench4_$TAG.err; echo rc4=$?; cut -c1-400 gpurun_out/bench4_$TAG.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python tools/profile_step.py --steps 5 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dyn_step -s 1 -c 1 -o gpurun_out/prof_$TAG python tools/profile_step.py --steps 2 > gpurun_out/ncu_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_asu -c 4 -o gpurun_out/prof_asu_$TAG python tools/profile_step.py --entry asuca_step --steps 1 > gpurun_out/ncu_asu_$TAG.log 2>&1
tail -n1 gpurun_out/ncu_$TAG.log; tail -n1 gpurun_out/ncu_asu_$TAG.log
