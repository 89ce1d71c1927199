"""Per-phase cycle breakdown of job 0 (TACOS_TRACE) for a config, under clusters 1 and 2.
usage: python tools/trace_phases.py CONFIG"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
CHILD = r'''
import os, sys; sys.path.insert(0, %r)
import paper_2304_05301_b200 as T, workloads as W
wl = W.config(%d)
t = T.Topology.from_workload_topology(wl.topo)
s = T.synthesize(t, wl.collective, wl.chunks_per_npu, wl.chunk_bytes, wl.n_seeds,
                 no_schedule=os.environ.get("NOSCHED") == "1")
print("T", s.result["T"])
''' % (ROOT, cfg)
names = ["PA", "bar1", "PB", "PM", "bar_pm", "PE-a", "bar2", "PE-b"]
for q in [int(x) for x in os.environ.get("QS", "1,2").split(",")]:
    out = os.path.join(ROOT, "gpurun_out", f"trace_c{cfg}_q{q}.txt")
    env = dict(os.environ, TACOS_CLUSTER=str(q), TACOS_TRACE=out)
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    print(f"cluster {q}:", r.stdout.strip()[-100:], r.stderr.strip()[-300:])
    rows = [list(map(int, l.split())) for l in open(out)]
    for rank in sorted(set(x[0] for x in rows)):
        rr = [x for x in rows if x[0] == rank]
        n = len(rr)
        tot = [sum(x[6 + i] for x in rr) for i in range(8)]
        all_ = sum(tot)
        print(f"  rank {rank}: events {n}, cycles/event {all_ / n:.0f}: " +
              " ".join(f"{nm}={tot[i] / n:.0f}" for i, nm in enumerate(names)) +
              (f" | slowest PM thread {sum(x[14] for x in rr) / n:.0f} record thread {sum(x[15] for x in rr) / n:.0f}"
               if len(rr[0]) > 15 else "") +
              (f" | walker max prologue {sum(x[16] for x in rr) / n:.0f} walk {sum(x[17] for x in rr) / n:.0f}"
               f" steps {sum(x[18] for x in rr) / n:.1f}" if len(rr[0]) > 18 else ""))
