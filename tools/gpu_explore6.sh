L=$PWD/paper_2304_05301_b200
for i in 1 2; do
for v in "" hoist t352; do
  if [ -n "$v" ]; then export TACOS_LIB=$L/libtacos_$v.so; else unset TACOS_LIB; fi
  timeout 120 python tools/time_search.py 3 0 50 2>&1 | tail -1
done; done
unset TACOS_LIB
for c in 2 5; do timeout 120 python tools/time_search.py $c 0 20 2>&1 | tail -1; done
TACOS_LIB=$L/libtacos_hoist.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
