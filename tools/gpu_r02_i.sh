# r02 call I: config 4 windowed -- cluster sizes, and a source-level ncu of the current loop.
python -c "from paper_2304_05301_b200 import build; build.build()"
for q in 4 5 6 8; do TACOS_CLUSTER=$q timeout 300 python tools/time_search.py 4 0 2; done > gpurun_out/r02i_c4_q.txt 2>&1; cat gpurun_out/r02i_c4_q.txt
python tools/time_search.py 4 0 1 > gpurun_out/r02i_c4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:greedy -c 1 -o gpurun_out/r02i_prof_c4w -f \
    python tools/time_search.py 4 0 1 > gpurun_out/r02i_ncu_c4w.log 2>&1; echo "ncu rc=$?"
