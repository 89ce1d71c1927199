# r02 call K: lazy have-row load in the windowed loop; parity + timing (configs 4, 5, 3).
python -c "from paper_2304_05301_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "windowed or hetero_mesh or config4_every" > gpurun_out/r02k_window.log 2>&1; echo "window rc=$?"; tail -2 gpurun_out/r02k_window.log
for c in 4 5 3 2; do timeout 300 python tools/time_search.py $c 0 5; done > gpurun_out/r02k_time.txt 2>&1; cat gpurun_out/r02k_time.txt
