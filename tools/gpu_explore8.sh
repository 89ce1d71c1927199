for q in 4 8; do TACOS_CLUSTER=$q timeout 200 python tools/time_search.py 4 1 2 2>&1 | tail -1; done
TACOS_CLUSTER=8 TACOS_THREADS=256 timeout 200 python tools/time_search.py 4 1 2 2>&1 | tail -1
TACOS_CLUSTER=8 TACOS_WORKLIST=0 timeout 200 python tools/time_search.py 4 1 2 2>&1 | tail -1
