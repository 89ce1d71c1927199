# r02 call F: windowed event loop -- parity (checked build first), then timing on config 4.
python -c "from paper_2304_05301_b200 import build; build.build()"
CK=paper_2304_05301_b200/libtacos_checked.so
TACOS_LIB=$CK timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "windowed or hetero_mesh" > gpurun_out/r02f_checked_window.log 2>&1; echo "checked window rc=$?"; tail -30 gpurun_out/r02f_checked_window.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "windowed or hetero_mesh or config4_every" --durations=5 > gpurun_out/r02f_window.log 2>&1; echo "window rc=$?"; tail -12 gpurun_out/r02f_window.log
for wdw in 1 0; do TACOS_WINDOW=$wdw timeout 300 python tools/time_search.py 4 0 3; done > gpurun_out/r02f_c4_time.txt 2>&1; cat gpurun_out/r02f_c4_time.txt
