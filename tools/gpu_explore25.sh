timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --no-cpu-baseline --no-baselines 2>&1 | tail -1 | cut -c1-250
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3b.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/ncu_launches.log 2>&1
grep -h "rs_uniform\|seg_starts" gpurun_out/launches_c3b.csv | head -4 | cut -c1-50,200-400
