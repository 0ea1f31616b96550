timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hfc.py tests/test_gpu_peer.py tests/test_gpu_tolerance.py -q -x -p no:cacheprovider -k "asuca or graph or tolerance or fma or variant or ab_variants" 2>&1 | tail -15
for r in 1 2; do
  for a in exact fma; do python tools/time_step.py 1581 1301 58 full $a 2>&1 | tail -1; done
done
python tools/time_step.py 1581 1301 58 asuca 2>&1 | tail -6
python tools/time_step.py 512 512 58 asuca 2>&1 | tail -6
