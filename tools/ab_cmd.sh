for r in 1 2; do
for ms in 20 100 1000; do
  echo -n "smi $ms: "; timeout 600 python bench.py --no-secondary --smi-ms $ms 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'], d['clocks']['samples'])"
done
done
