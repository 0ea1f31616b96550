# tall columns (65 < nz <= 129) through the fused kernels: parity, launches, memcheck
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "large or tall or golden" 2>&1 | tail -3
timeout 300 compute-sanitizer --tool memcheck --print-limit 3 python tools/debug_asuca.py 40 30 100 2>&1 | grep -v "Host Frame\|^=========         " | tail -3
timeout 300 compute-sanitizer --tool memcheck --print-limit 3 python tools/debug_tma.py 40 30 120 2>&1 | grep -v "Host Frame\|^=========         " | tail -3
for n in 58 100; do python tools/time_step.py 512 512 $n 2>&1 | tail -1; python tools/time_step.py 512 512 $n asuca 2>&1 | tail -5 | head -1; done
