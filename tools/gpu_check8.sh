for PD in 0 1; do TACOS_PRE_DRAW=$PD timeout 200 python tools/time_search.py 4 0 3 2>&1 | tail -1; done
for PD in 0 1; do TACOS_PRE_DRAW=$PD TACOS_LANES=8 timeout 200 python tools/time_search.py 4 0 3 2>&1 | tail -1; done
