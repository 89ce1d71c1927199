"""Per-phase cycle breakdown of the windowed event loop (TACOS_TRACE, job 0) for a config.
usage: python tools/trace_windows.py [CONFIG] [SEEDS]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
seeds = int(sys.argv[2]) if len(sys.argv) > 2 else 0
CHILD = r'''
import os, sys; sys.path.insert(0, %r)
import paper_2304_05301_b200 as T, workloads as W
wl = W.config(%d)
t = T.Topology.from_workload_topology(wl.topo)
s = T.synthesize(t, wl.collective, wl.chunks_per_npu, wl.chunk_bytes, %d or wl.n_seeds, no_schedule=True)
print("T", s.result["T"])
''' % (ROOT, cfg, seeds)
names = ["mark", "bar1", "list", "arrivals", "bar3", "done", "dest", "end+bar6"]
out = os.path.join(ROOT, "gpurun_out", f"trace_windows_c{cfg}.txt")
r = subprocess.run([sys.executable, "-c", CHILD], env=dict(os.environ, TACOS_TRACE=out), capture_output=True, text=True)
print(r.stdout.strip()[-100:], r.stderr.strip()[-300:])
rows = [list(map(int, l.split())) for l in open(out)]
for rank in sorted(set(x[0] for x in rows)):
    rr = [x for x in rows if x[0] == rank]
    n = len(rr)
    tot = [sum(x[6 + i] for x in rr) for i in range(8)]
    print(f"rank {rank}: windows {n}, events/window {sum(x[3] for x in rr) / n:.1f} (run {sum(x[4] for x in rr) / n:.1f}), "
          f"cycles/window {sum(tot) / n:.0f}: " + " ".join(f"{nm}={tot[i] / n:.0f}" for i, nm in enumerate(names)) +
          f" | group phase max {sum(x[14] for x in rr) / n:.0f} min {sum(x[15] for x in rr) / n:.0f}"
          f" | processed (dest, event) {sum(x[16] for x in rr) / n:.0f} walked links {sum(x[17] for x in rr) / n:.0f}")
