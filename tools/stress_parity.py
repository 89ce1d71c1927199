"""Randomized GPU-vs-oracle parity sweep (not part of the test suite): random strongly
connected graphs, costs, chunk counts, collectives, variants (link-first, one link cost =
lock-step loop, literal, relays, windowed wide rows) and forced cluster sizes (1-16); every mismatch is printed with its instance.
usage: python tools/stress_parity.py [N_CASES] [SEED]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_2304_05301_b200 as T  # noqa: E402
import workloads as W  # noqa: E402

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 12345)
T.load_library()
fails = 0
done = {}
skipped = 0
t0 = time.time()
for case in range(n_cases):
    mode = rng.choice(["plain", "plain", "uniform", "wide", "literal", "relay", "custom"])
    n = int(rng.integers(3, 24 if mode != "wide" else 14))
    m = int(rng.integers(n, min(n * (n - 1), 4 * n) + 1))
    alphas = tuple(int(x) for x in rng.integers(0, 20000, size=int(rng.integers(1, 5))))
    bws = tuple(int(x) for x in rng.choice([25, 50, 100, 200, 400], size=int(rng.integers(1, 4))))
    if mode == "uniform":  # one link cost: the lock-step loop (in-degree <= 8, <= 512 chunks)
        alphas, bws = alphas[:1], bws[:1]
    topo = W.random_strongly_connected(n, m, int(rng.integers(0, 2**31)), bws=bws, alphas=alphas)
    k = int(rng.integers(1, 6)) if mode != "wide" else -(-1100 // n) + int(rng.integers(0, 30))
    seeds = int(rng.integers(1, 6))
    base = int(rng.integers(0, 2**40))
    coll = str(rng.choice(["AG", "RS", "AR"]))
    nbytes = int(rng.choice([4096, 65536, 1 << 20]))
    env = {}
    if rng.random() < 0.3:
        env["TACOS_CLUSTER"] = str(int(rng.integers(1, 17)))
    if mode == "wide" and rng.random() < 0.5:
        env["TACOS_WIN_EV"] = str(int(rng.choice([1, 2, 5])))
    kw, okw = {}, {}
    if mode == "literal":
        kw["literal"] = okw["literal"] = True
    if mode in ("relay", "custom"):
        C = int(rng.integers(1, 40))
        pre_s, post_s = {}, {}
        for c in range(C):
            for x in rng.choice(n, int(rng.integers(1, 3)), replace=False).tolist():
                pre_s.setdefault(x, []).append(c)
            need = rng.choice(n, int(rng.integers(0, n + 1)), replace=False).tolist()
            for x in set(need) | set(x for x, cs in pre_s.items() if c in cs):
                post_s.setdefault(x, []).append(c)
        if mode == "custom":  # no relays: every NPU requires every chunk (R17)
            post_s = {x: list(range(C)) for x in range(n)}
        pre = oracle.bits_from_sets(n, C, pre_s)
        post = oracle.bits_from_sets(n, C, post_s)
        coll, k = "CUSTOM", 1
        kw.update(pre=pre, post=post, n_chunks=C)
        okw.update(pre=pre, post=post, n_chunks=C)
        if mode == "relay":
            kw["relay"] = okw["relay"] = True
    try:
        syn = oracle.synthesize(topo, k, nbytes, coll, [(base + s) % 2**64 for s in range(seeds)], **okw)
    except oracle.OracleError:  # a stall: skipped (counted)
        skipped += 1
        continue
    old = {kk: os.environ.get(kk) for kk in env}
    os.environ.update(env)
    try:
        t = T.Topology.from_workload_topology(topo)
        sch = T.synthesize(t, coll, k, nbytes, seeds, base, keep_seed_times=True, **kw)
        ok = (sch.result["T"] == syn.T and sch.sends.tobytes() == syn.sends.tobytes()
              and np.array_equal(sch.seed_times, np.asarray(syn.seed_times, dtype=np.uint64)))
        runs = list(syn.ag) + (list(syn.rs) if syn.rs is not syn.ag else [])
        ok = ok and (sch.result["visits"], sch.result["matches"], sch.result["events"]) == (
            sum(r.V for r in runs), sum(r.M for r in runs), sum(r.E for r in runs))
    except Exception as e:  # noqa: BLE001
        ok = False
        print("EXC", e)
    finally:
        for kk, v in old.items():
            if v is None:
                os.environ.pop(kk, None)
            else:
                os.environ[kk] = v
    done[mode] = done.get(mode, 0) + 1
    if not ok:
        fails += 1
        print(f"MISMATCH case {case}: mode={mode} n={n} m={m} k={k} coll={coll} seeds={seeds} base={base} "
              f"env={env} alphas={alphas} bws={bws}")
print(f"{n_cases} cases ({done}, {skipped} skipped as stalls), {fails} mismatches, {time.time() - t0:.0f} s")
sys.exit(1 if fails else 0)
