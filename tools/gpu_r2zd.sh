# bench with graph-replayed secondary configs; exact vs fma interleaved (sustained)
timeout 900 python bench.py --steps 100 --warmup 5 > gpurun_out/bench_r2zd.json 2> gpurun_out/bench_r2zd.err; tail -2 gpurun_out/bench_r2zd.err
python3 -c "
import json
d=json.load(open('gpurun_out/bench_r2zd.json'))
print(d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['tolerance_mode']['ms_per_step'])
for k,v in d['other_configs'].items(): print(k[:50], v['ms_per_step'], v['frac_of_measured_hbm'])
"
for r in 1 2; do for a in exact fma; do timeout 120 python tools/time_sustained.py $a 2>&1 | tail -1; done; done
