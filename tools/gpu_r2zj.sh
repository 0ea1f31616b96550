# the bench's ASUCA line (1 GPU; 2 ranks on one GPU through the decomposed scheme)
timeout 900 python bench.py --entry asuca_step --steps 10 --warmup 3 --no-secondary > gpurun_out/bench_asu.json 2> gpurun_out/bench_asu.err; tail -3 gpurun_out/bench_asu.err
cut -c1-2500 gpurun_out/bench_asu.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --entry asuca_step --steps 4 --warmup 3 --tile512 --one-gpu-test --no-secondary --trace > gpurun_out/bench_asu2.json 2> gpurun_out/bench_asu2.err; echo rc=$?; grep "bench rank 0" gpurun_out/bench_asu2.err | tail -4; cut -c1-400 gpurun_out/bench_asu2.json
