# debug the x-shared tendency pass: memcheck on a small grid (full report in gpurun_out/)
timeout 600 compute-sanitizer --tool memcheck python tools/debug_asuca.py 70 20 10 > gpurun_out/zq_memcheck.txt 2>&1
head -40 gpurun_out/zq_memcheck.txt
