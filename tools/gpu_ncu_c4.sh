ncu --set full --clock-control none --import-source on -k regex:greedy -c 1 -o gpurun_out/prof_c4 -f \
    python tools/time_search.py 4 1 1 > gpurun_out/ncu_c4.log 2>&1
tail -3 gpurun_out/ncu_c4.log
