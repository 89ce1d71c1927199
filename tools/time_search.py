"""Time the device search (tacos_plan_search) of a config under the current env.
usage: python tools/time_search.py CONFIG [no_schedule] [reps] [seeds]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2304_05301_b200 as T  # noqa: E402
import workloads as W  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
nosch = len(sys.argv) > 2 and sys.argv[2] == "1"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
wl = W.config(cfg)
if len(sys.argv) > 4:
    wl.n_seeds = int(sys.argv[4])
torch.cuda.set_device(0)
t = T.Topology.from_workload_topology(wl.topo)
pl = T.Plan(t, wl.collective, wl.chunks_per_npu, wl.chunk_bytes, wl.n_seeds, no_schedule=nosch)
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    pl.search(st)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    pl.search(st)
b.record()
torch.cuda.synchronize()
s = pl.stats(st)
env = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("TACOS_"))
print(f"config {cfg} no_schedule={int(nosch)} {env}: search {a.elapsed_time(b) / reps:.3f} ms  E={s['events']} M={s['matches']}")
