for i in 1 2; do timeout 120 python tools/time_search.py 3 0 50 2>&1 | tail -1; done
for c in 2 5; do timeout 120 python tools/time_search.py $c 0 20 2>&1 | tail -1; done
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "config3 or config2 or config5" 2>&1 | tail -1
QS=2 timeout 300 python tools/trace_phases.py 3
