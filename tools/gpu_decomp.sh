timeout 600 python -m pytest tests/test_gpu_decomp.py -m gpu -q -p no:cacheprovider 2>&1 | tail -5
