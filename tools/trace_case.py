"""Dump the event trace (TACOS_TRACE) of job 0 for a small hetero mesh under clusters 1 and 2."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys; sys.path.insert(0, %r)
import paper_2304_05301_b200 as T, workloads as W
t = T.Topology.from_workload_topology(W.mesh2d(16, 16, 200, 100))
try:
    s = T.synthesize(t, "AG", 1, 128 << 10, 1)
    print("T", s.result["T"])
except Exception as e:
    print("err", e)
''' % ROOT
for q in (1, 2):
    out = os.path.join(ROOT, "gpurun_out", f"trace_q{q}.txt")
    env = dict(os.environ, TACOS_CLUSTER=str(q), TACOS_TRACE=out)
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    print(q, r.stdout[-300:], r.stderr[-300:])
