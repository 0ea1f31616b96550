timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python tools/debug_asuca.py 128 96 58 2>&1 | grep -v 'Host Frame\|^=========         in ' | tail -12
timeout 2000 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hfc.py tests/test_gpu_peer.py tests/test_gpu_tolerance.py -q -p no:cacheprovider -k "asuca or graph or tolerance or fma or variant or ab_variants" 2>&1 | tail -15
python tools/time_step.py 1581 1301 58 asuca 2>&1 | tail -6
python tools/time_step.py 512 512 58 asuca 2>&1 | tail -6
