timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for i in 1 2; do
timeout 120 python tools/time_search.py 3 0 50 2>&1 | tail -1
TACOS_LIB=$PWD/paper_2304_05301_b200/libtacos_head.so timeout 120 python tools/time_search.py 3 0 50 2>&1 | tail -1
done
for c in 2 5; do timeout 120 python tools/time_search.py $c 0 20 2>&1 | tail -1; TACOS_LIB=$PWD/paper_2304_05301_b200/libtacos_head.so timeout 120 python tools/time_search.py $c 0 20 2>&1 | tail -1; done
