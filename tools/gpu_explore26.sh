timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "all_seeds or edge or forced" 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3c.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/ncu_launches.log 2>&1
python - <<'PY'
import csv
from collections import defaultdict
rows=[r for r in csv.reader(open('gpurun_out/launches_c3c.csv')) if len(r)>10]
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value")
agg=defaultdict(list)
for r in rows[1:]: agg[r[ki].split('(')[0]].append(float(r[vi].replace(',',''))/1000)
for k,v in sorted(agg.items(), key=lambda x:-sum(x[1])): print(f"{k[:60]:60s} {len(v):3d} {sum(v)/len(v):8.2f} us")
PY
