for q in 4 5 6 7; do TACOS_DEBUG_OCC=1 TACOS_CLUSTER=$q timeout 200 python tools/time_search.py 4 1 2 2>&1 | grep -E "max active|search" | head -2; done
TACOS_CLUSTER=6 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "hetero or config4 or all_seeds" 2>&1 | tail -1
TACOS_CLUSTER=3 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "hetero or all_seeds or forced" 2>&1 | tail -1
