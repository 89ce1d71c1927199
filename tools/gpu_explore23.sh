for i in 1 2; do
timeout 120 python tools/time_search.py 3 0 50 2>&1 | tail -1
TACOS_LANES=2 timeout 120 python tools/time_search.py 3 0 50 2>&1 | tail -1
done
TACOS_LANES=2 timeout 120 python tools/time_search.py 2 0 20 2>&1 | tail -1
timeout 120 python tools/time_search.py 2 0 20 2>&1 | tail -1
TACOS_LANES=2 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
TACOS_LANES=2 QS=2 timeout 300 python tools/trace_phases.py 3
