timeout 900 python bench.py --steps 100 --warmup 5 > gpurun_out/bench_r2ze.json 2> gpurun_out/bench_r2ze.err; tail -2 gpurun_out/bench_r2ze.err
python3 -c "
import json
d=json.load(open('gpurun_out/bench_r2ze.json'))
print(d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['tolerance_mode'])
"
timeout 900 python -m pytest tests/test_gpu_peer.py -q -p no:cacheprovider -k "bench_multi_rank" 2>&1 | tail -2
