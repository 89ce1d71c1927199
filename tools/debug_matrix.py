"""Run cases under several env settings in subprocesses and compare with the oracle.
usage: python tools/debug_matrix.py"""
import itertools
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = {
    "mesh16_hetero_k8": "W.mesh2d(16, 16, 200, 100), 8",
    "mesh16_uniform_k8": "W.mesh2d(16, 16, 100, 100), 8",
    "torus8x8x8_k1": "W.torus([8, 8, 8]), 1",
    "torus16x16_k1": "W.torus([16, 16]), 1",
    "mesh16_hetero_k1": "W.mesh2d(16, 16, 200, 100), 1",
}
CHILD = r'''
import sys, json
sys.path.insert(0, %r)
import paper_2304_05301_b200 as T, workloads as W
topo, k = %s
t = T.Topology.from_workload_topology(topo)
try:
    s = T.synthesize(t, "AG", k, 128 << 10, 2, keep_seed_times=True)
    print(json.dumps({"times": [int(x) for x in s.seed_times], "V": s.result["visits"]}))
except Exception as e:
    print(json.dumps({"err": str(e)[:120]}))
'''

if __name__ == "__main__":
    sys.path.insert(0, ROOT)
    import oracle
    import workloads as W
    for name, expr in CASES.items():
        topo, k = eval(expr)
        ref = oracle.synthesize(topo, k, 128 << 10, "AG", [0, 1])
        print(name, "oracle", [g.T for g in ref.ag], sum(g.V for g in ref.ag), flush=True)
        for cl, ln in itertools.product([1, 2], [1, 4, 16]):
            env = dict(os.environ, TACOS_CLUSTER=str(cl), TACOS_LANES=str(ln))
            out = subprocess.run([sys.executable, "-c", CHILD % (ROOT, expr)], env=env, capture_output=True, text=True,
                                 timeout=300)
            print(f"   cluster={cl} lanes={ln}:", out.stdout.strip()[-200:], out.stderr.strip()[-200:], flush=True)
