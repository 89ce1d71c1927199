timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --no-cpu-baseline --no-baselines 2>&1 | tail -1 | cut -c1-330
python bench.py --config 2 --no-cpu-baseline --no-baselines 2>&1 | tail -1 | cut -c1-330
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
