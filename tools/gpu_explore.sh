# Phase traces and search timings of configs 3 and 4 under cluster / lane overrides.
QS=2 timeout 300 python tools/trace_phases.py 3
QS=4 timeout 600 python tools/trace_phases.py 4
for q in 2 4 8; do TACOS_CLUSTER=$q timeout 300 python tools/time_search.py 4 1 2 2>&1 | tail -1; done
TACOS_LANES=2 timeout 300 python tools/time_search.py 3 0 20 2>&1 | tail -1
timeout 300 python tools/time_search.py 3 0 20 2>&1 | tail -1
timeout 300 python tools/time_search.py 3 1 20 2>&1 | tail -1
