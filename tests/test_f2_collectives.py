"""Row f2 (general pre/post collectives with relays, rooted collectives,
multi-tenant merges): the oracle against what the paper and the mathematics
fix.  CPU only (the library's host-side verifier tacos_eval is used as an
independent checker of the oracle's schedules).

Pins:
  * P:L116 (Fig. NonAwareCollective) / P:L155-161 (Fig. CollectiveOnTEN):
    Scatter on a 4-NPU unidirectional ring takes 3 steps; the exhaustive
    optimum with unrestricted relays is 3 steps and best-of-S greedy reaches it.
  * Broadcast of one chunk floods: every NPU receives the chunk at its hop
    distance from the root, so T = eccentricity(root) * w on homogeneous
    topologies (the greedy sends the one chunk on every free link whose source
    holds it and whose destination lacks it).
  * Reduce is the time reversal of Broadcast on G^T, Gather that of
    Scatter (same T; mirror o mirror = id).
  * R22 relays: every relay send moves its chunk one hop closer to an NPU that
    requires it; no NPU receives a chunk twice; the schedule passes tacos_eval.
"""
from collections import deque

import numpy as np
import pytest

import oracle
import oracle.collectives as OC
import workloads as W
from bruteforce import optimum
from verify import check, clean

MiB = 1 << 20


@pytest.fixture(scope="module")
def T():
    from paper_2304_05301_b200 import build

    build.build()
    import paper_2304_05301_b200 as T

    T.load_library()
    return T


def hops_from(n, src, dst, root):
    out = [[] for _ in range(n)]
    for s, d in zip(src.tolist(), dst.tolist()):
        out[s].append(d)
    dist = [-1] * n
    dist[root] = 0
    q = deque([root])
    while q:
        x = q.popleft()
        for y in out[x]:
            if dist[y] < 0:
                dist[y] = dist[x] + 1
                q.append(y)
    return dist


def masks(bits):
    """N x W u32 rows -> per-NPU python int bitmasks (for the brute force)."""
    return [sum(int(v) << (32 * i) for i, v in enumerate(row)) for row in np.asarray(bits)]


def test_scatter_uni_ring4_three_steps():
    """"Scatter on a 4-NPU uni ring takes 3 steps" -- the exhaustive
    optimum (relays unrestricted) is 3 w, every greedy seed is >= 3 w, and the
    best of 32 seeds reaches it."""
    topo = W.uni_ring(4)
    w = oracle.link_cost(500, 100, MiB)
    C, pre, post = OC.named_bits("SCATTER", 4, 1, 0)
    links = [(int(s), int(d), 1) for s, d in zip(topo.src, topo.dst)]
    assert optimum(4, links, masks(pre), masks(post), t_max=8, relays=True) == 3
    assert optimum(4, links, masks(pre), masks(post), t_max=8, relays=False) is None  # relays are required
    syn = oracle.synthesize(topo, 1, MiB, "SCATTER", list(range(32)), root=0)
    assert syn.T == 3 * w
    assert all(int(t) >= 3 * w for t in syn.seed_times)


@pytest.mark.parametrize("shape", ["uni4", "bi5", "path4"])
def test_gather_scatter_vs_bruteforce(shape):
    """Greedy with shortest-path relays never beats the exhaustive optimum with
    unrestricted relays (small instances, w = 1)."""
    topo = {"uni4": W.uni_ring(4), "bi5": W.bi_ring(5), "path4": W.path(4)}[shape]
    n = topo.n_npus
    links = [(int(s), int(d), 1) for s, d in zip(topo.src, topo.dst)]
    w = oracle.link_cost(500, 100, MiB)
    for kind in ("SCATTER", "GATHER"):
        C, pre, post = OC.named_bits(kind, n, 1, 0)
        opt = optimum(n, links, masks(pre), masks(post), t_max=12, relays=True)
        assert opt is not None
        syn = oracle.synthesize(topo, 1, MiB, kind, list(range(8)), root=0)
        assert syn.T >= opt * w


@pytest.mark.parametrize("shape,root", [("mesh6", 2), ("mesh6", 17), ("torus44", 5), ("bi7", 3), ("hyper16", 0)])
def test_broadcast_is_eccentricity(shape, root):
    topo = {"mesh6": W.mesh2d(6, 6), "torus44": W.torus([4, 4]), "bi7": W.bi_ring(7),
            "hyper16": W.hypercube(4)}[shape]
    w = oracle.link_cost(int(topo.alpha_ns[0]), int(topo.bw[0]), MiB)
    ecc = max(hops_from(topo.n_npus, topo.src, topo.dst, root))
    for coll in ("BROADCAST", "REDUCE"):
        syn = oracle.synthesize(topo, 1, MiB, coll, [0, 1, 2], root=root)
        assert syn.T == ecc * w
        assert all(int(t) == ecc * w for t in syn.seed_times)  # every seed floods the same way
        assert syn.sends.shape[0] == topo.n_npus - 1


def test_reduce_gather_are_mirrors():
    """REDUCE / GATHER = mirror of BROADCAST / SCATTER on G^T (asymmetric
    graph: searched on G^T with sigma = 1; symmetric: same-seed mirror)."""
    for topo in (W.random_strongly_connected(10, 24, 7, bws=(25, 50, 100), alphas=(0, 500)), W.mesh2d(4, 4)):
        w = oracle.link_costs(topo, MiB)
        rev = oracle.reverse_links(topo.src, topo.dst, w)
        for kind, fwd in (("REDUCE", "BROADCAST"), ("GATHER", "SCATTER")):
            syn = oracle.synthesize(topo, 1, MiB, kind, [3, 4], root=1)
            C, pre, post = OC.named_bits(fwd, topo.n_npus, 1, 1)
            allow = OC.relay_allow(topo.n_npus, topo.dst if rev is None else topo.src,
                                   topo.src if rev is None else topo.dst, C, pre, post) if fwd == "SCATTER" else None
            a, b, sig = (topo.dst, topo.src, 1) if rev is None else (topo.src, topo.dst, 0)
            runs = [oracle.greedy(topo.n_npus, a, b, w, C, 0, s, sig, pre, post, allow=allow) for s in (3, 4)]
            best = min(runs, key=lambda r: r.T)
            assert syn.T == best.T
            back = oracle.mirror(syn.sends, syn.T, topo.src, topo.dst, rev)
            assert np.array_equal(oracle.canonical(back), oracle.canonical(best.sends))


@pytest.mark.parametrize("case", ["scatter_mesh", "gather_torus", "gather_rand_asym", "custom_path", "tenants"])
def test_relay_invariants_and_verifier(T, case):
    if case == "scatter_mesh":
        topo, kind, k, root = W.mesh2d(4, 5), "SCATTER", 2, 7
    elif case == "gather_torus":
        topo, kind, k, root = W.torus([3, 4]), "GATHER", 1, 0
    elif case == "gather_rand_asym":  # G^T search; relays in flight at the end leave the schedule
        topo, kind, k, root = W.random_strongly_connected(10, 24, 7, bws=(25, 50, 100), alphas=(0, 500)), "GATHER", 1, 3
    elif case == "custom_path":
        topo, kind, k, root = W.path(6), "CUSTOM", 1, 0
    else:
        topo, kind, k, root = W.mesh2d(4, 4), "TENANTS", 1, 0
    n = topo.n_npus
    t = T.Topology.from_workload_topology(topo)
    if kind == "CUSTOM":  # end NPUs exchange: 0 -> 5 and 5 -> 0 through 4 relays
        C = 2
        pre = oracle.bits_from_sets(n, C, {0: [0], 5: [1]})
        post = oracle.bits_from_sets(n, C, {0: [0, 1], 5: [0, 1]})
        syn = oracle.synthesize(topo, 1, MiB, "CUSTOM", list(range(4)), pre=pre, post=post, n_chunks=C, relay=True)
        rep = T.evaluate(t, syn.sends, "CUSTOM", 1, MiB, pre=pre, post=post, n_chunks=C, relay=True)
        assert syn.T == 5 * oracle.link_cost(500, 100, MiB)  # both chunks walk the 5 hops at once
    elif kind == "TENANTS":
        C, pre, post, first = OC.multi_tenant(n, [("BROADCAST", 2, 1), ("REDUCE", 9, 1), ("AG", 0, 1)])
        syn = oracle.synthesize(topo, 1, MiB, "CUSTOM", list(range(4)), pre=pre, post=post, n_chunks=C, relay=True)
        rep = T.evaluate(t, syn.sends, "CUSTOM", 1, MiB, pre=pre, post=post, n_chunks=C, relay=True)
        C2, pre2, post2, first2 = T.multi_tenant(n, [("BROADCAST", 2, 1), ("REDUCE", 9, 1), ("AG", 0, 1)])
        assert (C2, first2) == (C, first) and np.array_equal(pre2, pre) and np.array_equal(post2, post)
    else:
        syn = oracle.synthesize(topo, k, MiB, kind, list(range(4)), root=root)
        rep = T.evaluate(t, syn.sends, kind, k, MiB, root=root)
        C, pre, post = OC.named_bits(kind if kind == "SCATTER" else OC.dual(kind), n, k, root)
    assert rep["n_violations"] == 0, rep
    # the independent replay of tests/verify.py (structural rules; relays follow R22, not the
    # link-first maximality): a GATHER is mirrored back onto G^T, where it is a Scatter
    sends = syn.sends
    fwd = kind != "GATHER"
    w = oracle.link_costs(topo, MiB)
    sets = lambda bits: [{c for c in range(C) if (int(bits[x, c >> 5]) >> (c & 31)) & 1} for x in range(n)]
    if fwd:
        v = check(n, topo.src, topo.dst, w, sends, sets(pre), sets(post), greedy=False)
    else:
        back = oracle.mirror(sends, syn.T, topo.src, topo.dst, None)
        v = check(n, topo.dst, topo.src, w, back, sets(pre), sets(post), greedy=False)
    assert clean(v), v
    a, b = (topo.src, topo.dst) if fwd else (topo.dst, topo.src)
    seen = set()
    for e in sends.tolist():
        c, s, d = e[0], e[1], e[2]
        if not fwd:
            s, d = d, s
        assert (d, c) not in seen
        seen.add((d, c))
        if not (int(post[d, c >> 5]) >> (c & 31)) & 1:
            req = [x for x in range(n) if (int(post[x, c >> 5]) >> (c & 31)) & 1 and not (int(pre[x, c >> 5]) >> (c & 31)) & 1]
            dist = OC.hop_distance_to(n, a, b, req)
            assert dist[d] + 1 == dist[s]
    required = int(sum(bin(int(v)).count("1") for v in (post & ~pre).ravel()))
    assert sends.shape[0] >= required


def test_multi_tenant_table6_shape():
    """P:L478 Table VI scenario (6 x 6 mesh; Broadcast from NPU 2, Reduce to NPU 17,
    All-Gather) synthesizes, meets every tenant's postcondition and is no faster
    than its slowest tenant alone (tenants share the links)."""
    topo = W.mesh2d(6, 6)
    n = 36
    C, pre, post, first = OC.multi_tenant(n, [("BROADCAST", 2, 1), ("REDUCE", 17, 1), ("AG", 0, 1)])
    syn = oracle.synthesize(topo, 1, MiB, "CUSTOM", list(range(8)), pre=pre, post=post, n_chunks=C, relay=True)
    alone = oracle.synthesize(topo, 1, MiB, "AG", list(range(8)))
    ecc2 = max(hops_from(n, topo.src, topo.dst, 2))
    w = oracle.link_cost(500, 100, MiB)
    assert syn.T >= ecc2 * w
    lb_ag = max(max(hops_from(n, topo.src, topo.dst, x)) for x in range(n)) * w  # diameter
    assert syn.T >= lb_ag
    assert alone.T >= lb_ag
    got = np.zeros_like(pre)
    got |= pre
    for e in syn.sends.tolist():
        got[e[2], e[0] >> 5] |= np.uint32(1 << (e[0] & 31))
    assert np.all((post & ~got) == 0)


@pytest.mark.parametrize("n,tenants", [
    (36, [("BROADCAST", 2, 1), ("REDUCE", 17, 1), ("AG", 0, 1)]),
    (16, [("SCATTER", 3, 2), ("GATHER", 15, 1), ("BROADCAST", 0, 5)]),
    (9, [("AG", 0, 3), ("AG", 0, 1), ("REDUCE", 8, 2), ("SCATTER", 4, 1)]),
    (2, [("GATHER", 1, 7)]),
])
def test_multi_tenant_abi_matches_oracle(T, n, tenants):
    """tacos_multi_tenant (C ABI) builds the same merged pre/post as the oracle's
    plain-numpy merge (Table VI; R23)."""
    C, pre, post, first = OC.multi_tenant(n, tenants)
    C2, pre2, post2, first2 = T.multi_tenant(n, tenants)
    assert (C2, first2) == (C, first)
    assert np.array_equal(pre2, pre) and np.array_equal(post2, post)


def test_multi_tenant_abi_errors(T):
    with pytest.raises(T.TacosError) as e:
        T.multi_tenant(4, [("BROADCAST", 4, 1)])
    assert e.value.code == T.TACOS_E_INVALID_ARG
    with pytest.raises(T.TacosError) as e:
        T.multi_tenant(4, [("AG", 0, 0)])
    assert e.value.code == T.TACOS_E_INVALID_ARG
    with pytest.raises(T.TacosError) as e:
        T.multi_tenant(1024, [("AG", 0, 8), ("AG", 0, 9)])
    assert e.value.code == T.TACOS_E_OVERFLOW
