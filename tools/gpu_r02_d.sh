# r02 call D: GPU suite after the staged plan upload, bounds-checked build on the sanitize cases and the
# parity suite (compute-sanitizer is closed on this pool), e2e breakdown, full ncu of config 3's search.
python -c "from paper_2304_05301_b200 import build; build.build()"
python paper_2304_05301_b200/build.py --variant checked -DTACOS_CHECKED=1 > /dev/null
python -m pytest tests -m gpu -x -q > gpurun_out/r02d_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02d_pytest_gpu.log
export CK=paper_2304_05301_b200/libtacos_checked.so
TACOS_LIB=$CK python tools/sanitize_cases.py > gpurun_out/r02d_checked_cases.txt 2>&1; echo "checked cases rc=$?"; tail -3 gpurun_out/r02d_checked_cases.txt
TACOS_LIB=$CK python -m pytest tests/test_gpu_parity.py tests/test_gpu_f2.py -x -q -k "not config4_every" > gpurun_out/r02d_checked_pytest.log 2>&1; echo "checked pytest rc=$?"; tail -3 gpurun_out/r02d_checked_pytest.log
python tools/host_breakdown.py 3 > gpurun_out/r02d_host_breakdown_c3.txt 2>&1; cat gpurun_out/r02d_host_breakdown_c3.txt
python tools/time_search.py 3 0 2 > gpurun_out/r02d_c3_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:greedy -s 2 -c 1 -o gpurun_out/r02d_prof_c3 -f \
    python tools/time_search.py 3 0 2 > gpurun_out/r02d_ncu_c3.log 2>&1; echo "ncu rc=$?"
