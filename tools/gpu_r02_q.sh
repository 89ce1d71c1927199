# r02 call Q: window walk with per-vector reductions + one lane scan; parity + config 4 timing.
python -c "from paper_2304_05301_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_random_graphs.py -x -q -m gpu -k "windowed or hetero_mesh or config4_every or custom_pre_post" > gpurun_out/r02q_window.log 2>&1; echo "window rc=$?"; tail -2 gpurun_out/r02q_window.log
timeout 300 python tools/time_search.py 4 0 3 > gpurun_out/r02q_c4.txt 2>&1; cat gpurun_out/r02q_c4.txt
