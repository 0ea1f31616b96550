for r in 1 2; do
for ms in 20 100 1000; do
  echo -n "smi $ms: "; HFB_BENCH_SMI_MS=$ms timeout 600 python bench.py --no-secondary 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'], d['clocks']['samples'])"
done
done
