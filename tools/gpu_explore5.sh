WPF=$PWD/paper_2304_05301_b200/libtacos_wpf.so
timeout 200 python tools/time_search.py 4 1 2 2>&1 | tail -1
TACOS_LIB=$WPF timeout 200 python tools/time_search.py 4 1 2 2>&1 | tail -1
timeout 120 python tools/time_search.py 3 0 50 2>&1 | tail -1
TACOS_LIB=$WPF timeout 120 python tools/time_search.py 3 0 50 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
TACOS_LIB=$WPF timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "config4 or mesh or wide or k64 or k512" 2>&1 | tail -2
QS=4 timeout 600 python tools/trace_phases.py 4
