# r02 call J: windowed loop with a shared destination queue + register-cached source arrivals.
python -c "from paper_2304_05301_b200 import build; build.build()"
CK=paper_2304_05301_b200/libtacos_checked.so
TACOS_LIB=$CK timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "windowed or hetero_mesh" > gpurun_out/r02j_checked_window.log 2>&1; echo "checked window rc=$?"; tail -2 gpurun_out/r02j_checked_window.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "windowed or hetero_mesh or config4_every" > gpurun_out/r02j_window.log 2>&1; echo "window rc=$?"; tail -2 gpurun_out/r02j_window.log
for q in 6 5; do TACOS_CLUSTER=$q timeout 300 python tools/time_search.py 4 0 3; done > gpurun_out/r02j_c4_time.txt 2>&1; cat gpurun_out/r02j_c4_time.txt
