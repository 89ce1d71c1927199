for Q in 1 2 4 8; do TACOS_CLUSTER=$Q timeout 200 python tools/time_search.py 4 0 3 2>&1 | tail -1; done
TACOS_CLUSTER=4 QS=4 timeout 300 python tools/trace_phases.py 4 2>&1 | tail -5
timeout 120 python tools/time_search.py 3 0 20 2>&1 | tail -1
