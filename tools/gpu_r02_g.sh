# r02 call G: config 5 with the compact live-list walk, config 4 windowed ncu (source-level stalls).
python -c "from paper_2304_05301_b200 import build; build.build()"
python -m pytest tests/test_gpu_parity.py -x -q -k "config_parity_all_seeds or edge_cases or batch_mixed or forced_cluster" > gpurun_out/r02g_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02g_pytest.log
python tools/time_search.py 5 0 20 > gpurun_out/r02g_c5_time.txt 2>&1; cat gpurun_out/r02g_c5_time.txt
python tools/time_search.py 4 0 1 > gpurun_out/r02g_c4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:greedy -c 1 -o gpurun_out/r02g_prof_c4w -f \
    python tools/time_search.py 4 0 1 > gpurun_out/r02g_ncu_c4w.log 2>&1; echo "ncu rc=$?"
