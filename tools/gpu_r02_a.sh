# r02 call A: host info, full GPU test suite (incl. config-4 every-seed parity), ncu of config 4's search.
nproc; free -g | head -2
python -c "from paper_2304_05301_b200 import build; build.build()"
python -m pytest tests -m gpu -x -q > gpurun_out/r02a_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r02a_pytest_gpu.log
python tools/time_search.py 4 0 1 > gpurun_out/r02a_c4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:greedy -c 1 -o gpurun_out/r02a_prof_c4 -f \
    python tools/time_search.py 4 0 1 > gpurun_out/r02a_ncu_c4.log 2>&1; echo "ncu rc=$?"
tail -2 gpurun_out/r02a_c4_plain.log gpurun_out/r02a_ncu_c4.log
