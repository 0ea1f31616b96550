timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hfc.py tests/test_checked.py -q -p no:cacheprovider -k "asuca or checked or unset or raises or division or valid" 2>&1 | tail -6
python tools/time_step.py 1581 1301 58 asuca 2>&1 | tail -6
for r in 1 2; do
  for L in paper_1710_08616_b200/libhfb.so ab/libhfb_doc.so ab/libhfb_o1.so; do
    for a in exact fma; do echo -n "$L "; HFB_LIB=$L timeout 120 python tools/time_sustained.py $a 2>&1 | tail -1; done
  done
done
