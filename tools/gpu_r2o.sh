# the ASUCA scheme on decomposed contexts (peer transport) + regression of the exchange
# refactor (peer, in-process groups)
timeout 1500 python -m pytest tests/test_gpu_peer.py tests/test_gpu_decomp.py -q -p no:cacheprovider -x 2>&1 | tail -8
