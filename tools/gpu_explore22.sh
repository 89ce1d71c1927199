L=$PWD/paper_2304_05301_b200
timeout 200 python tools/time_search.py 4 1 2 2>&1 | tail -1
TACOS_LIB=$L/libtacos_hpf384.so timeout 200 python tools/time_search.py 4 1 2 2>&1 | tail -1
TACOS_LIB=$L/libtacos_hpf.so timeout 200 python tools/time_search.py 4 1 2 2>&1 | tail -1
TACOS_LIB=$L/libtacos_t320.so timeout 200 python tools/time_search.py 4 1 2 2>&1 | tail -1
TACOS_LIB=$L/libtacos_hpf384.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "hetero or config4 or forced" 2>&1 | tail -1
