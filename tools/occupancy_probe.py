"""Does a second resident CTA per SM pay?  Times the search of an 8x8x4 torus AG (k = 1,
one CTA of ~100 KB shared memory per seed, so two fit on an SM) at S = 148 and 296 seeds."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2304_05301_b200 as T  # noqa: E402
import workloads as W  # noqa: E402

torch.cuda.set_device(0)
t = T.Topology.from_workload_topology(W.torus([8, 8, 4]))
st = torch.cuda.current_stream().cuda_stream
for S in (74, 148, 222, 296, 444):
    pl = T.Plan(t, "AG", 1, 1 << 20, S, no_schedule=True)
    for _ in range(3):
        pl.search(st)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        pl.search(st)
    b.record()
    torch.cuda.synchronize()
    print(f"S={S}: search {a.elapsed_time(b) / 10:.3f} ms", flush=True)
