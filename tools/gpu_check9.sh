python -m pytest tests -m gpu -x -q -k "not config4_full_size" > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
TACOS_LANES=2 python -m pytest tests/test_gpu_parity.py -x -q -k "not config4_full_size" 2>&1 | tail -1
for c in 3 2 5 4; do timeout 200 python tools/time_search.py $c 0 5 2>&1 | tail -1; done
