"""Where the end-to-end time of one synthesis goes (config 3 by default): topology load
(host CSR + H2D), plan build, search, emission, D2H of the schedule; medians of 20 calls.
usage: python tools/host_breakdown.py [CONFIG] [SEEDS]"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2304_05301_b200 as T  # noqa: E402
import workloads as W  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
wl = W.config(cfg)
S = int(sys.argv[2]) if len(sys.argv) > 2 else wl.n_seeds
torch.cuda.set_device(0)
T.load_library()
st = torch.cuda.Stream()
sh = st.cuda_stream
p, keep = T.make_params(wl.collective, wl.chunks_per_npu, wl.chunk_bytes, S)
tt = T.Topology.from_workload_topology(wl.topo)
n = T.max_sends(tt, p)
host = torch.empty(n * 32, dtype=torch.uint8).pin_memory()
dev = torch.empty(n * 32, dtype=torch.uint8, device="cuda")
parts = {k: [] for k in ("topology", "plan", "search", "emit", "d2h", "total_split", "synthesize_into")}
for i in range(25):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    t1 = T.Topology.from_workload_topology(wl.topo)
    ta = time.perf_counter()
    pl = T.Plan(t1, wl.collective, wl.chunks_per_npu, wl.chunk_bytes, S)
    tb = time.perf_counter()
    pl.search(sh)
    st.synchronize()
    tc = time.perf_counter()
    pl.emit(dev.data_ptr(), n, sh)
    st.synchronize()
    td = time.perf_counter()
    with torch.cuda.stream(st):
        host.copy_(dev, non_blocking=True)
    st.synchronize()
    te = time.perf_counter()
    del pl
    t2 = T.Topology.from_workload_topology(wl.topo)
    tf = time.perf_counter()
    T.synthesize_into(t2, p, host.data_ptr(), n, sh)
    tg = time.perf_counter()
    if i >= 5:
        for k, v in (("topology", ta - t0), ("plan", tb - ta), ("search", tc - tb), ("emit", td - tc), ("d2h", te - td),
                     ("total_split", te - t0), ("synthesize_into", tg - tf)):
            parts[k].append(v * 1e3)
print(f"config {cfg}, {S} seeds, {n} sends ({n * 32 / 1e6:.1f} MB)")
for k, v in parts.items():
    print(f"  {k:16s} median {statistics.median(v):8.3f} ms   min {min(v):8.3f} ms")
