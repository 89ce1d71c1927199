# GPU iteration: parity tests (quick subset unless FULL=1), then search timings
if [ "$FULL" = "1" ]; then python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; else
python -m pytest tests -m gpu -x -q -k "not config4_full_size" > gpurun_out/pytest_gpu.log 2>&1; fi
tail -3 gpurun_out/pytest_gpu.log
for c in 2 3 5 4; do timeout 120 python tools/time_search.py $c 0 10 2>&1 | tail -1; done
