set -x
for L in 1 2 4; do for Q in 1 2 4; do for PD in 0 1; do
TACOS_LANES=$L TACOS_CLUSTER=$Q TACOS_PRE_DRAW=$PD timeout 60 python tools/time_search.py 3 0 20 2>&1 | tail -1
done; done; done
for L in 1 2 4 8; do TACOS_LANES=$L timeout 60 python tools/time_search.py 2 0 20 2>&1 | tail -1; done
