for c in 1 2 4 8; do echo "chunk $c"; for s in "1581 1301 58" "512 512 58"; do HFB_DIFF_CHUNK=$c timeout 120 python tools/time_step.py $s diffusion 2>&1 | tail -1; done; done
