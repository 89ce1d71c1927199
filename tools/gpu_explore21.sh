for q in 4 5 6; do TACOS_CLUSTER=$q timeout 200 python tools/time_search.py 4 1 2 2>&1 | tail -1; done
