# r02 call H: windowed loop with per-destination event skipping -- parity (checked build, then plain), timing.
python -c "from paper_2304_05301_b200 import build; build.build()"
CK=paper_2304_05301_b200/libtacos_checked.so
TACOS_LIB=$CK timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "windowed or hetero_mesh" > gpurun_out/r02h_checked_window.log 2>&1; echo "checked window rc=$?"; tail -3 gpurun_out/r02h_checked_window.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "windowed or hetero_mesh or config4_every" > gpurun_out/r02h_window.log 2>&1; echo "window rc=$?"; tail -3 gpurun_out/r02h_window.log
for wdw in 1 0; do TACOS_WINDOW=$wdw timeout 300 python tools/time_search.py 4 0 3; done > gpurun_out/r02h_c4_time.txt 2>&1; cat gpurun_out/r02h_c4_time.txt
