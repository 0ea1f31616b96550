# final tree: the full GPU suite, smoke, the bench line, the reference arm
TAG=r2zl
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 100 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -2 gpurun_out/bench_$TAG.err
python3 -c "
import json
d=json.load(open('gpurun_out/bench_$TAG.json'))
print(d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['tolerance_mode']['ms_per_step'], d['tolerance_mode']['exact_ms_per_step_same_state'])
for k,v in d['other_configs'].items(): print(k[:50], v['ms_per_step'], v['frac_of_measured_hbm'])
"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; tail -2 gpurun_out/bench_ref_$TAG.err
