python -m pytest tests -m gpu -x -q -k "not config4_full_size" > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for c in 3 2 5 4; do for PD in 0 1; do TACOS_PRE_DRAW=$PD timeout 120 python tools/time_search.py $c 0 10 2>&1 | tail -1; done; done
QS=2 python tools/trace_phases.py 3 2>&1 | tail -3
