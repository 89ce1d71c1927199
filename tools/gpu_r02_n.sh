# r02 call N: live-visit counts (config 4, 3, 5), config 2 cluster sizes.
python -c "from paper_2304_05301_b200 import build; build.build()"
python - <<'PY' > gpurun_out/r02n_lv.txt 2>&1
import sys; sys.path.insert(0, ".")
import torch, paper_2304_05301_b200 as T, workloads as W
torch.cuda.set_device(0)
for c in (3, 5, 4, 2):
    wl = W.config(c)
    t = T.Topology.from_workload_topology(wl.topo)
    pl = T.Plan(t, wl.collective, wl.chunks_per_npu, wl.chunk_bytes, wl.n_seeds)
    st = torch.cuda.current_stream().cuda_stream
    pl.search(st)
    s = pl.stats(st)
    print(c, {k: s[k] for k in ("visits", "live_visits", "matches", "dest_events", "events")})
PY
cat gpurun_out/r02n_lv.txt
for q in 1 2; do TACOS_CLUSTER=$q python tools/time_search.py 2 0 20; done > gpurun_out/r02n_c2_q.txt 2>&1; cat gpurun_out/r02n_c2_q.txt
