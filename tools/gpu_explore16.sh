timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for i in 1 2; do
timeout 120 python tools/time_search.py 3 0 50 2>&1 | tail -1
TACOS_CLUSTER=4 timeout 120 python tools/time_search.py 3 0 50 2>&1 | tail -1
done
TACOS_CLUSTER=4 TACOS_THREADS=256 timeout 120 python tools/time_search.py 3 0 50 2>&1 | tail -1
TACOS_CLUSTER=4 TACOS_THREADS=160 timeout 120 python tools/time_search.py 3 0 50 2>&1 | tail -1
timeout 200 python tools/time_search.py 4 1 2 2>&1 | tail -1
TACOS_CLUSTER=4 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
