for q in 4 8; do TACOS_DEBUG_OCC=1 TACOS_CLUSTER=$q timeout 200 python tools/time_search.py 4 1 1 2>&1 | grep -m1 "max active"; done
TACOS_DEBUG_OCC=1 TACOS_CLUSTER=4 timeout 200 python tools/time_search.py 3 1 1 2>&1 | grep -m1 "max active"
TACOS_DEBUG_OCC=1 timeout 200 python tools/time_search.py 3 1 1 2>&1 | grep -m1 "max active"
