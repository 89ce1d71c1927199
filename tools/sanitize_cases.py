"""Small synthesis cases for compute-sanitizer (memcheck / racecheck / synccheck), each
checked against the oracle: configs 1-2, forced cluster splits Q = 2 / 4 / 8 (DSMEM mirror
pushes, cluster barriers), the lock-step loop, the paper-literal kernel (f1), a relay collective (f2), the
global-row (config-4 shape) path and the RS sort / uniform emitters.
usage: python tools/sanitize_cases.py [quick]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CASES = [
    # (name, env, topology expr, collective, k, seeds, extra kwargs)
    ("config1_ag", {}, "W.config(1).topo", "AG", 1, 4, {}),
    ("config2_ar", {}, "W.config(2).topo", "AR", 4, 4, {}),
    ("torus4x4_q2", {"TACOS_CLUSTER": "2"}, "W.torus([4, 4])", "AR", 2, 3, {}),
    ("torus8x8x8_q4", {"TACOS_CLUSTER": "4"}, "W.torus([8, 8, 8])", "AR", 1, 2, {}),
    ("hetero_mesh8x8_q8", {"TACOS_CLUSTER": "8"}, "W.mesh2d(8, 8, 200, 100)", "AR", 3, 2, {}),
    ("mesh8x16_k64_global_rows", {}, "W.mesh2d(8, 16, 200, 100)", "AR", 64, 2, {}),
    ("rand_asym_rs", {}, "W.random_strongly_connected(9, 20, 5, bws=(25, 50, 100), alphas=(0, 500))", "RS", 2, 3, {}),
    ("literal_torus4x4", {}, "W.torus([4, 4])", "AR", 2, 3, {"literal": True}),
    # lock-step loop: double-buffered rows pushed as 16-byte DSMEM stores, compact link state
    ("lockstep_torus8x8x8_q2", {}, "W.torus([8, 8, 8])", "AR", 1, 3, {}),
    ("lockstep_uni_ring9_q3", {"TACOS_CLUSTER": "3"}, "W.uni_ring(9)", "AR", 3, 3, {}),
    ("lockstep_torus4x4_q8", {"TACOS_CLUSTER": "8"}, "W.torus([4, 4])", "AG", 2, 3, {}),
    ("scatter_mesh6", {}, "W.mesh2d(6, 6)", "SCATTER", 1, 3, {"root": 2}),
]

CHILD = r'''
import sys; sys.path.insert(0, {root!r})
import torch, oracle, workloads as W, paper_2304_05301_b200 as T
torch.cuda.set_device(0)
topo = {topo}
kw = {kw!r}
t = T.Topology.from_workload_topology(topo)
sch = T.synthesize(t, {coll!r}, {k}, 1 << 20, {seeds}, keep_seed_times=True, **kw)
syn = oracle.synthesize(topo, {k}, 1 << 20, {coll!r}, list(range({seeds})), **kw)
assert sch.result["T"] == syn.T and sch.sends.tobytes() == syn.sends.tobytes(), {name!r}
print({name!r}, "ok T =", syn.T)
'''


def main():
    failed = 0
    for name, env, topo, coll, k, seeds, kw in CASES:
        code = CHILD.format(root=ROOT, topo=topo, kw=kw, coll=coll, k=k, seeds=seeds, name=name)
        e = dict(os.environ, **env)
        r = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True)
        sys.stdout.write(r.stdout)
        if r.returncode:
            failed += 1
            sys.stdout.write(f"{name} FAILED rc={r.returncode}\n{r.stderr[-2000:]}\n")
    print("failed cases:", failed)
    return 1 if failed else 0


if __name__ == "__main__":
    sys.exit(main())
