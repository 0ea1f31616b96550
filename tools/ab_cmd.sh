for o in 0 1 2; do HFB_TILE_ORDER=$o timeout 100 python tools/debug_tma.py 70 45 58 | tr '\n' ' '; echo; done
for r in 1 2; do
  for o in 0 1 2; do
    echo -n "[order $o] "; HFB_TILE_ORDER=$o timeout 120 python tools/time_step.py 512 512 58 2>&1 | tail -1
    echo -n "[order $o] "; HFB_TILE_ORDER=$o timeout 120 python tools/time_step.py 1581 1301 58 2>&1 | tail -1
  done
done
for o in 0 1 2; do HFB_TILE_ORDER=$o ncu --metrics dram__bytes.sum -k regex:k_dyn_step_ws -s 3 -c 1 python tools/time_step.py 512 512 58 2>&1 | grep dram__bytes; done
