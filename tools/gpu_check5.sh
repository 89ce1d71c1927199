python -m pytest tests -m gpu -x -q -k "not config4_full_size" > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for L in 1 2; do for PD in 0 1; do TACOS_LANES=$L TACOS_PRE_DRAW=$PD timeout 120 python tools/time_search.py 3 0 20 2>&1 | tail -1; done; done
for c in 2 5; do for PD in 0 1; do TACOS_PRE_DRAW=$PD timeout 120 python tools/time_search.py $c 0 10 2>&1 | tail -1; done; done
TACOS_PRE_DRAW=0 QS=2 python tools/trace_phases.py 3 2>&1 | tail -2
