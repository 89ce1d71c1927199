"""tacos_eval's greedy-rule checks (NOT_MAXIMAL, NOT_SHORTER_FIRST; SURVEY §8(c) P11,
P:L253 maximal matching per event, P:L263-264 shorter-link-first) against the
independent replay in tests/verify.py, on oracle schedules (clean) and on
schedules broken on purpose (each rule violated once).  CPU only: tacos_eval is
host code of the library."""
import numpy as np
import pytest

import oracle
import workloads as W
from verify import ag_sets, check, clean

MiB = 1 << 20


@pytest.fixture(scope="module")
def T():
    from paper_2304_05301_b200 import build

    build.build()
    import paper_2304_05301_b200 as T

    T.load_library()
    return T


CASES = {
    "uni5": (W.uni_ring(5), 1),
    "torus44_k2": (W.torus([4, 4]), 2),
    "mesh6_hetero_k3": (W.mesh2d(6, 6, 200, 100), 3),
    "rand9_asym_k2": (W.random_strongly_connected(9, 22, 3, bws=(25, 50, 100), alphas=(0, 500)), 2),
    "hybrid_fail": (W.remove_undirected_links(W.switch_hypercube_hybrid(4, 8, 20, 25), 0.05, 2)[0], 1),
    "config2": (W.config(2).topo, 4),
}


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("coll", ["AG", "RS", "AR"])
def test_oracle_schedules_obey_greedy_rules(T, name, coll):
    topo, k = CASES[name]
    syn = oracle.synthesize(topo, k, 256 << 10, coll, [0, 1, 2])
    t = T.Topology.from_workload_topology(topo)
    rep = T.evaluate(t, syn.sends, coll, k, 256 << 10)
    assert rep["n_violations"] == 0, rep
    if coll == "AG":  # the independent replay agrees
        w = oracle.link_costs(topo, 256 << 10)
        pre, post = ag_sets(topo.n_npus, k)
        assert clean(check(topo.n_npus, topo.src, topo.dst, w, syn.sends, pre, post))


def _e5(T):
    """Fig. HeterogeneousGreedy(a): links l0 = 1->2 (w 2), l1 = 0->2 (w 1);
    chunk 0 held by NPUs 0 and 1, required by 2."""
    topo = W.Topology(3, np.array([1, 0], np.int32), np.array([2, 2], np.int32), np.array([1, 0], np.uint32),
                      np.array([2**31] * 2, np.uint32))
    pre = oracle.bits_from_sets(3, 1, {0: [0], 1: [0]})
    post = oracle.bits_from_sets(3, 1, {0: [0], 1: [0], 2: [0]})
    return topo, pre, post


def test_costlier_link_first_is_flagged(T):
    topo, pre, post = _e5(T)
    t = T.Topology.from_workload_topology(topo)
    good = np.zeros(1, dtype=T.SEND_DTYPE)
    good[0] = (0, 0, 2, 1, 0, 1)
    bad = np.zeros(1, dtype=T.SEND_DTYPE)
    bad[0] = (0, 1, 2, 0, 0, 2)  # the 2-cost link took chunk 0 while the 1-cost link idled
    ok = T.evaluate(t, good, "CUSTOM", 1, 1, pre=pre, post=post, n_chunks=1)
    assert ok["n_violations"] == 0
    rep = T.evaluate(t, bad, "CUSTOM", 1, 1, pre=pre, post=post, n_chunks=1)
    assert rep["not_shorter_first"] == 1 and rep["n_violations"] == 1 and rep["first_index"] == 1
    v = check(3, topo.src, topo.dst, [2, 1], bad, [{0}, {0}, set()], [{0}, {0}, {0}])
    assert len(v["not_shorter_first"]) == 1 and len(v.get("not_maximal", [])) == 0


@pytest.mark.parametrize("name", ["uni5", "torus44_k2", "mesh6_hetero_k3"])
def test_delayed_send_is_not_maximal(T, name):
    """Move one last-step AG send (a delivery no other send depends on) to start at T:
    still a valid schedule, but its link idled with an unclaimed candidate."""
    topo, k = CASES[name]
    nb = 256 << 10
    syn = oracle.synthesize(topo, k, nb, "AG", [0])
    s = syn.sends.copy()
    T_ag = int(s["t_end"].max())
    i = int(np.flatnonzero(s["t_end"] == T_ag)[0])
    w = int(s[i]["t_end"] - s[i]["t_start"])
    s[i]["t_start"] = T_ag
    s[i]["t_end"] = T_ag + w
    t = T.Topology.from_workload_topology(topo)
    rep = T.evaluate(t, s, "AG", k, nb)
    # the idle link flagged first is an in-link of the delayed send's destination
    assert rep["not_maximal"] >= 1 and int(topo.dst[rep["first_index"]]) == int(s[i]["dst"])
    assert rep["n_violations"] == rep["not_maximal"] + rep["not_shorter_first"]
    wv = oracle.link_costs(topo, nb)
    pre, post = ag_sets(topo.n_npus, k)
    v = check(topo.n_npus, topo.src, topo.dst, wv, s, pre, post)
    assert len(v["not_maximal"]) >= 1


def test_literal_and_relay_schedules_skip_greedy_rules(T):
    """R21 / R22 follow other rules: their schedules are checked structurally only."""
    topo = W.uni_ring(4)
    t = T.Topology.from_workload_topology(topo)
    syn = oracle.synthesize(topo, 1, MiB, "SCATTER", list(range(8)), root=0)
    rep = T.evaluate(t, syn.sends, "SCATTER", 1, MiB, root=0)
    assert rep["n_violations"] == 0
