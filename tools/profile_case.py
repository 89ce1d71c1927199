"""Run one best-of-S synthesis of a config through the C ABI (for ncu /
compute-sanitizer captures).  usage: python tools/profile_case.py CONFIG [SEEDS] [REPEAT]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2304_05301_b200 as T  # noqa: E402
import workloads as W  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
seeds = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rep = int(sys.argv[3]) if len(sys.argv) > 3 else 2
wl = W.config(cfg)
S = seeds or wl.n_seeds
torch.cuda.set_device(0)
t = T.Topology.from_workload_topology(wl.topo)
for i in range(rep):
    s = T.synthesize(t, wl.collective, wl.chunks_per_npu, wl.chunk_bytes, S)
torch.cuda.synchronize()
print(f"config {cfg}: T={s.result['T']} seed={s.result['seed']} V={s.result['visits']} M={s.result['matches']}")
