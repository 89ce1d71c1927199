TACOS_LIB=$PWD/paper_2304_05301_b200/libtacos_head.so TACOS_CLUSTER=4 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "all_seeds" 2>&1 | tail -2
TACOS_CLUSTER=2 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "all_seeds" 2>&1 | tail -2
TACOS_WORKLIST=1 TACOS_CLUSTER=4 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "all_seeds" 2>&1 | tail -2
