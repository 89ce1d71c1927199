for i in 1 2; do
timeout 120 python tools/time_search.py 3 0 50 2>&1 | tail -1
TACOS_LIB=$PWD/paper_2304_05301_b200/libtacos_hreg.so timeout 120 python tools/time_search.py 3 0 50 2>&1 | tail -1
done
for th in 288 320 384 416; do TACOS_THREADS=$th timeout 120 python tools/time_search.py 3 0 50 2>&1 | tail -1; done
TACOS_LIB=$PWD/paper_2304_05301_b200/libtacos_hreg.so timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "config3 or config2 or config5" 2>&1 | tail -1
TACOS_LIB=$PWD/paper_2304_05301_b200/libtacos_hreg.so QS=2 timeout 300 python tools/trace_phases.py 3
