"""Property-based cases on random strongly connected digraphs (hypothesis).

CPU part: every schedule the oracle produces on a random graph, with random
link costs (alpha, bw), chunks per NPU and seed, passes the independent replay
checker (exactly-once delivery, held at departure
P:L266-267, link intervals disjoint P:L146, maximality and shorter-link-first
at every event P:L253) and respects the per-node lower bound.

GPU part: the CUDA path through the C ABI against the oracle on the same random
instances, bit-exact (schedule, per-seed times, counters), for AG / RS / AR and
both greedy variants (link-first R1/R4 and paper-literal R21).
"""
import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import oracle
import workloads as W
from verify import ag_sets, check, clean


@st.composite
def instances(draw, max_n=9):
    n = draw(st.integers(2, max_n))
    n_links = draw(st.integers(n, n * (n - 1))) if n > 2 else 2
    gseed = draw(st.integers(0, 2**31 - 1))
    bws = tuple(draw(st.lists(st.sampled_from([1, 7, 25, 50, 100, 400]), min_size=1, max_size=3)))
    alphas = tuple(draw(st.lists(st.sampled_from([0, 1, 500, 1500, 20000]), min_size=1, max_size=3)))
    topo = W.random_strongly_connected(n, n_links, gseed, bws=bws, alphas=alphas)
    k = draw(st.sampled_from([1, 2, 3, 5, 17]))
    nbytes = draw(st.sampled_from([1, 4096, 1 << 20, 3 << 20]))
    seed = draw(st.integers(0, 2**64 - 1))
    return topo, k, nbytes, seed


def _bound(topo, w, k):
    """Smallest T at which every node's in-links could have carried its C - k
    missing chunks (in-link l moves at most floor(T / w_l) of them by T)."""
    C = topo.n_npus * k
    best = 0
    for d in range(topo.n_npus):
        ws = [int(w[l]) for l in range(topo.n_links) if int(topo.dst[l]) == d]
        lo, hi = 0, (C - k) * max(ws)
        while lo < hi:
            mid = (lo + hi) // 2
            if sum(mid // q for q in ws) >= C - k:
                hi = mid
            else:
                lo = mid + 1
        best = max(best, lo)
    return best


@settings(max_examples=60, deadline=None, derandomize=True, suppress_health_check=[HealthCheck.too_slow])
@given(instances(), st.booleans())
def test_oracle_schedules_valid_on_random_graphs(inst, literal):
    topo, k, nbytes, seed = inst
    w = oracle.link_costs(topo, nbytes)
    res = oracle.greedy(topo.n_npus, topo.src, topo.dst, w, topo.n_npus * k, k, seed, literal=literal)
    rep = check(topo.n_npus, topo.src, topo.dst, w, res.sends, *ag_sets(topo.n_npus, k), greedy=not literal)
    # literal variant (R21): replaced sends are cancelled, so only the final schedule's validity is checked
    assert clean(rep), {a: b[:5] for a, b in rep.items() if a != "T"}
    assert rep["T"] == res.T
    assert len(res.sends) == topo.n_npus * k * (topo.n_npus - 1) == res.M - res.X
    assert res.T >= _bound(topo, w, k)


@pytest.fixture(scope="module")
def T():
    import torch

    assert torch.cuda.is_available()
    from paper_2304_05301_b200 import build

    build.build()
    import paper_2304_05301_b200 as T

    T.load_library()
    return T


@pytest.mark.gpu
@settings(max_examples=150, deadline=None, derandomize=True, suppress_health_check=[HealthCheck.too_slow,
                                                                 HealthCheck.function_scoped_fixture])
@given(instances(max_n=16), st.sampled_from(["AG", "RS", "AR"]), st.booleans(), st.integers(1, 9))
def test_gpu_parity_on_random_graphs(T, inst, coll, literal, seeds):
    from test_gpu_parity import assert_parity, oracle_literal_stats

    topo, k, nbytes, base = inst
    base %= 2**32
    syn = oracle.synthesize(topo, k, nbytes, coll, [base + s for s in range(seeds)], literal=literal)
    t = T.Topology.from_workload_topology(topo)
    sch = T.synthesize(t, coll, k, nbytes, seeds, base, keep_seed_times=True, literal=literal)
    assert_parity(syn, sch, coll)
    rep = T.evaluate(t, sch.sends, coll, k, nbytes, literal=literal)
    assert rep["n_violations"] == 0, rep
    if literal:
        assert sch.result["cancelled"] == oracle_literal_stats(syn)


@st.composite
def custom_sets(draw, n):
    """Random pre/post over C chunks: every chunk has >= 1 holder, post is pre
    plus random requirers (relays make every such instance reachable, R22)."""
    C = draw(st.integers(1, 40))
    pre, post = {}, {}
    for c in range(C):
        holders = draw(st.lists(st.integers(0, n - 1), min_size=1, max_size=2, unique=True))
        need = draw(st.lists(st.integers(0, n - 1), max_size=n, unique=True))
        for x in holders:
            pre.setdefault(x, []).append(c)
        for x in set(holders) | set(need):
            post.setdefault(x, []).append(c)
    return C, pre, post


@settings(max_examples=80, deadline=None, derandomize=True, suppress_health_check=[HealthCheck.too_slow])
@given(instances(max_n=14), st.data())
def test_oracle_custom_relays_complete_on_random_graphs(inst, data):
    """R22: with relays along shortest paths to every requirer that lacks a
    chunk, every CUSTOM instance on a strongly connected graph completes (no
    stall) and its schedule is valid: links exist, durations, disjoint link
    intervals, departures only with held chunks, post met exactly once."""
    topo, _, nbytes, seed = inst
    n = topo.n_npus
    C, pre_s, post_s = data.draw(custom_sets(n))
    pre, post = oracle.bits_from_sets(n, C, pre_s), oracle.bits_from_sets(n, C, post_s)
    syn = oracle.synthesize(topo, 1, nbytes, "CUSTOM", [seed % 2**64], pre=pre, post=post, n_chunks=C, relay=True)
    w = oracle.link_costs(topo, nbytes)
    pre_sets = [set(pre_s.get(x, [])) for x in range(n)]
    post_sets = [set(post_s.get(x, [])) for x in range(n)]
    rep = check(n, topo.src, topo.dst, w, syn.sends, pre_sets, post_sets, greedy=False)
    assert clean(rep), {a: b[:5] for a, b in rep.items() if a != "T"}
    assert rep["T"] == syn.T


@pytest.mark.gpu
@settings(max_examples=80, deadline=None, derandomize=True, suppress_health_check=[HealthCheck.too_slow,
                                                                                   HealthCheck.function_scoped_fixture])
@given(instances(max_n=14), st.sampled_from(["BROADCAST", "REDUCE", "SCATTER", "GATHER", "CUSTOM"]),
       st.integers(1, 6), st.data())
def test_gpu_rooted_and_relay_parity_on_random_graphs(T, inst, coll, seeds, data):
    """Row f2 on random graphs: rooted collectives from a random root and random
    CUSTOM pre/post with relays, GPU vs oracle bit-exact, every schedule accepted
    by tacos_eval."""
    from test_gpu_f2 import check as f2_check

    topo, k, nbytes, _ = inst
    n = topo.n_npus
    root = data.draw(st.integers(0, n - 1))
    if coll == "CUSTOM":
        C, pre_s, post_s = data.draw(custom_sets(n))
        pre, post = oracle.bits_from_sets(n, C, pre_s), oracle.bits_from_sets(n, C, post_s)
        f2_check(T, topo, coll, 1, seeds, pre=pre, post=post, n_chunks=C, relay=True, nbytes=nbytes)
    else:
        f2_check(T, topo, coll, min(k, 5), seeds, root=root, nbytes=nbytes)


@pytest.mark.gpu
@settings(max_examples=40, deadline=None, derandomize=True, suppress_health_check=[HealthCheck.too_slow,
                                                                                   HealthCheck.function_scoped_fixture])
@given(instances(max_n=10), st.integers(1, 4), st.data())
def test_gpu_multi_tenant_parity_on_random_graphs(T, inst, seeds, data):
    """R23 on random graphs: 1-3 concurrent tenants (AG / Broadcast / Scatter /
    Gather / Reduce, random roots, 1-2 chunks each) merged into one CUSTOM
    pre/post with relays; GPU vs oracle bit-exact, accepted by tacos_eval, and
    the merge itself equals oracle.collectives.multi_tenant."""
    import oracle.collectives as OC
    from test_gpu_f2 import check as f2_check

    topo, _, nbytes, _ = inst
    n = topo.n_npus
    tenants = data.draw(st.lists(st.tuples(st.sampled_from(["AG", "BROADCAST", "SCATTER", "GATHER", "REDUCE"]),
                                           st.integers(0, n - 1), st.integers(1, 2)), min_size=1, max_size=3))
    C, pre, post, first = T.multi_tenant(n, tenants)
    C_o, pre_o, post_o, first_o = OC.multi_tenant(n, tenants)
    assert (C, list(first)) == (C_o, list(first_o))
    assert np.array_equal(np.asarray(pre, np.uint32).ravel(), np.asarray(pre_o, np.uint32).ravel())
    assert np.array_equal(np.asarray(post, np.uint32).ravel(), np.asarray(post_o, np.uint32).ravel())
    f2_check(T, topo, "CUSTOM", 1, seeds, pre=pre, post=post, n_chunks=C, relay=True, nbytes=nbytes)


@settings(max_examples=40, deadline=None, derandomize=True, suppress_health_check=[HealthCheck.too_slow])
@given(instances(max_n=8), st.integers(1, 4))
def test_oracle_inversion_on_random_graphs(inst, seeds):
    """P12 on random graphs (symmetric or not): the AR splits into an RS half
    ending at T_RS and an AG half starting there; the RS half mirrored back
    (c, b->a, T-t1, T-t0) replays as a valid All-Gather on G^T, mirroring twice
    is the identity, and the AG half shifted to 0 is a valid greedy All-Gather."""
    topo, k, nbytes, seed = inst
    n = topo.n_npus
    syn = oracle.synthesize(topo, k, nbytes, "AR", [(seed + s) % 2**64 for s in range(seeds)])
    w = oracle.link_costs(topo, nbytes)
    rs = syn.sends[syn.sends["t_end"] <= syn.T_rs]
    ag = syn.sends[syn.sends["t_start"] >= syn.T_rs]
    assert len(rs) + len(ag) == len(syn.sends) == 2 * n * k * (n - 1)
    assert syn.T == syn.T_rs + syn.T_ag
    back = oracle.mirror(rs, syn.T_rs, topo.src, topo.dst, None)
    gt = W.transpose(topo)
    rep = check(n, gt.src, gt.dst, w, back, *ag_sets(n, k), greedy=False)
    assert clean(rep), {a: b[:5] for a, b in rep.items() if a != "T"}
    assert rep["T"] == syn.T_rs
    twice = oracle.mirror(back, syn.T_rs, gt.src, gt.dst, None)
    assert np.array_equal(oracle.canonical(twice), oracle.canonical(rs))
    ag0 = ag.copy()
    ag0["t_start"] -= np.uint64(syn.T_rs)
    ag0["t_end"] -= np.uint64(syn.T_rs)
    rep2 = check(n, topo.src, topo.dst, w, ag0, *ag_sets(n, k))
    assert clean(rep2), {a: b[:5] for a, b in rep2.items() if a != "T"}


@st.composite
def wide_instances(draw):
    """Random graphs for the windowed loop: in-degree <= 8 (register path), C = N k >= 1025
    chunks (more than two lanes per row), several link costs, random window cut."""
    n = draw(st.integers(3, 12))
    n_links = draw(st.integers(n, min(n * (n - 1), 3 * n)))
    gseed = draw(st.integers(0, 2**31 - 1))
    alphas = tuple(draw(st.lists(st.integers(0, 30000), min_size=1, max_size=6)))
    bws = tuple(draw(st.lists(st.sampled_from([25, 50, 100, 200]), min_size=1, max_size=3)))
    topo = W.random_strongly_connected(n, n_links, gseed, bws=bws, alphas=alphas)
    k = -(-1025 // n) + draw(st.integers(0, 40))
    seed = draw(st.integers(0, 2**40))
    win_ev = draw(st.sampled_from(["1", "3", "256"]))
    return topo, k, seed, win_ev


@pytest.mark.gpu
@settings(max_examples=40, deadline=None, derandomize=True, suppress_health_check=[HealthCheck.too_slow,
                                                                HealthCheck.function_scoped_fixture])
@given(wide_instances(), st.sampled_from(["AG", "RS", "AR"]), st.integers(1, 4))
def test_gpu_windowed_loop_parity_on_random_graphs(T, inst, coll, seeds):
    """The windowed event loop (several link costs, wide rows) against the oracle on random
    graphs, bit-exact, with windows cut after 1, 3 or 256 events."""
    import os

    from test_gpu_parity import assert_parity

    topo, k, base, win_ev = inst
    if np.bincount(topo.dst, minlength=topo.n_npus).max() > 8:
        return
    nbytes = 64 << 10
    syn = oracle.synthesize(topo, k, nbytes, coll, [base + s for s in range(seeds)])
    t = T.Topology.from_workload_topology(topo)
    old = os.environ.get("TACOS_WIN_EV")
    os.environ["TACOS_WIN_EV"] = win_ev
    try:
        sch = T.synthesize(t, coll, k, nbytes, seeds, base, keep_seed_times=True)
    finally:
        if old is None:
            os.environ.pop("TACOS_WIN_EV", None)
        else:
            os.environ["TACOS_WIN_EV"] = old
    assert_parity(syn, sch, coll)
