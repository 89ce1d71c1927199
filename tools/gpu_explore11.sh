for q in 1 2 4; do TACOS_CLUSTER=$q timeout 120 python tools/time_search.py 2 0 20 2>&1 | tail -1; done
for q in 1 2; do TACOS_CLUSTER=$q timeout 120 python tools/time_search.py 5 0 10 2>&1 | tail -1; done
timeout 120 python tools/time_search.py 3 0 50 2>&1 | tail -1
