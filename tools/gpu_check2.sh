python -m pytest tests/test_gpu_f2.py -x -q > gpurun_out/f2.log 2>&1; tail -3 gpurun_out/f2.log
TACOS_LANES=2 python -m pytest tests/test_gpu_parity.py -x -q -k "not config4_full_size" > gpurun_out/lanes2.log 2>&1; tail -3 gpurun_out/lanes2.log
for L in 1 2; do for PD in 0 1; do TACOS_LANES=$L TACOS_PRE_DRAW=$PD timeout 60 python tools/time_search.py 3 0 20 2>&1 | tail -1; done; done
TACOS_LANES=2 timeout 60 python tools/time_search.py 2 0 20 2>&1 | tail -1
TACOS_LANES=2 timeout 60 python tools/time_search.py 5 0 10 2>&1 | tail -1
