"""GPU parity for row f2: rooted collectives (BROADCAST / REDUCE / SCATTER /
GATHER), CUSTOM pre/post with relays (R22) and multi-tenant merges (R23), the
CUDA path through the C ABI against the CPU oracle, element by element: the
winning time and seed, every seed's time, the counters V / D / M / E and the
schedule record by record.  Every schedule is also checked by tacos_eval."""
import numpy as np
import pytest

import oracle
import oracle.collectives as OC
import workloads as W

pytestmark = pytest.mark.gpu
MiB = 1 << 20


@pytest.fixture(scope="module")
def T():
    import torch

    assert torch.cuda.is_available()
    from paper_2304_05301_b200 import build

    build.build()
    import paper_2304_05301_b200 as T

    T.load_library()
    return T


def stats(syn):
    runs = list(syn.ag) + (list(syn.rs) if syn.rs is not syn.ag else [])
    return (sum(r.V for r in runs), sum(r.D for r in runs), sum(r.M for r in runs), sum(r.E for r in runs))


def check(T, topo, coll, k, seeds, root=0, pre=None, post=None, n_chunks=0, relay=False, nbytes=MiB):
    syn = oracle.synthesize(topo, k, nbytes, coll, list(range(seeds)), pre=pre, post=post,
                            n_chunks=n_chunks or None, relay=relay, root=root)
    t = T.Topology.from_workload_topology(topo)
    sch = T.synthesize(t, coll, k, nbytes, seeds, 0, keep_seed_times=True, pre=pre, post=post, n_chunks=n_chunks,
                       relay=relay, root=root)
    r = sch.result
    assert r["status"] == 0
    assert r["T"] == syn.T, (r["T"], syn.T)
    assert r["seed"] == syn.seed
    assert np.array_equal(sch.seed_times, np.asarray(syn.seed_times, dtype=np.uint64))
    assert (r["visits"], r["dest_events"], r["matches"], r["events"]) == stats(syn)
    assert sch.sends.shape == syn.sends.shape
    assert sch.sends.tobytes() == syn.sends.tobytes()
    rep = T.evaluate(t, sch.sends, coll, k, nbytes, pre=pre, post=post, n_chunks=n_chunks, root=root, relay=relay)
    assert rep["n_violations"] == 0, rep
    return syn, sch


@pytest.mark.parametrize("coll", ["BROADCAST", "REDUCE", "SCATTER", "GATHER"])
@pytest.mark.parametrize("shape", ["uni4", "mesh6", "torus44_k2", "rand10_asym"])
def test_rooted_collectives(T, coll, shape):
    topo, k, root, seeds = {
        "uni4": (W.uni_ring(4), 1, 0, 32),
        "mesh6": (W.mesh2d(6, 6), 1, 2 if coll in ("BROADCAST", "SCATTER") else 17, 8),
        "torus44_k2": (W.torus([4, 4]), 2, 5, 8),
        "rand10_asym": (W.random_strongly_connected(10, 24, 7, bws=(25, 50, 100), alphas=(0, 500)), 1, 3, 8),
    }[shape]
    check(T, topo, coll, k, seeds, root=root)


def test_scatter_uni_ring_three_steps(T):
    """Scatter on a 4-NPU uni ring: 3 steps (best of 32 seeds)."""
    syn, sch = check(T, W.uni_ring(4), "SCATTER", 1, 32, root=0)
    assert sch.result["T"] == 3 * oracle.link_cost(500, 100, MiB)


def test_scatter_wide_rows(T):
    """C = 512 chunks (4 vectors per lane) and C = 2048 on an 8 x 8 mesh."""
    check(T, W.mesh2d(8, 8), "SCATTER", 8, 4, root=27)
    check(T, W.mesh2d(8, 8), "GATHER", 32, 2, root=0)


def test_custom_relay_exchange(T):
    topo = W.path(6)
    C = 2
    pre = oracle.bits_from_sets(6, C, {0: [0], 5: [1]})
    post = oracle.bits_from_sets(6, C, {0: [0, 1], 5: [0, 1]})
    check(T, topo, "CUSTOM", 1, 4, pre=pre, post=post, n_chunks=C, relay=True)


def test_multi_tenant_table6(T):
    """P:L478 Table VI scenario: 6 x 6 mesh, Broadcast from NPU 2, Reduce to NPU 17
    (as a Gather of partials, R23) and All-Gather at once."""
    topo = W.mesh2d(6, 6)
    C, pre, post, _ = T.multi_tenant(36, [("BROADCAST", 2, 1), ("REDUCE", 17, 1), ("AG", 0, 1)])
    check(T, topo, "CUSTOM", 1, 16, pre=pre, post=post, n_chunks=C, relay=True)


def test_relay_plan_sharded(T):
    """Seed-sharded plans (multi-GPU shape) agree with the one-call path on a relay collective."""
    topo = W.mesh2d(5, 5)
    t = T.Topology.from_workload_topology(topo)
    full = T.synthesize(t, "SCATTER", 1, MiB, 8, 0, root=12)
    keys = []
    for off in (0, 4):
        pl = T.Plan(t, "SCATTER", 1, MiB, 4, 0, off, root=12)
        pl.search(0)
        keys.append(int(pl.best_keys_tensor()[0].item()))
    best = min(keys)
    assert best == T.make_key(full.result["T"], full.result["seed"])
