# One GPU: bench (config 3), then the launch list and one full ncu capture of the search kernel.
set -x
python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
tail -1 gpurun_out/bench_c3.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv \
    python bench.py --steps 3 --warmup 3 > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:greedy -s 3 -c 1 -o gpurun_out/prof_c3_bench -f \
    python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
