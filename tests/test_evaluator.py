"""Continuous-time evaluator and Ring / Direct baselines of the library (SURVEY
§8 row f3), against the plain rational-arithmetic reference in
oracle/evaluate.py and the numbers PAPER.md prints for them.  CPU only."""
import numpy as np
import pytest

import oracle
import oracle.evaluate as OE
import workloads as W

MiB = 1 << 20


@pytest.fixture(scope="module")
def T():
    from paper_2304_05301_b200 import build

    build.build()
    import paper_2304_05301_b200 as T

    T.load_library()
    return T


def test_paper_motivation_ratios(T):
    """P:L107 + P:L120 (Fig. ResultMotivationCollective, 100 NPUs, alpha = 0.5 us,
    100 GB/s, All-Reduce): "Ring ... 12.88x faster than Direct" on the 100-NPU
    Ring and Ring "99x slower" than Direct on the 100-NPU FullyConnected
    topology.  The Ring and Direct baselines evaluated in continuous time
    reproduce both printed ratios (any chunk size)."""
    for nb in (MiB, 64 << 10):
        ring = T.Topology.from_workload_topology(W.bi_ring(100))
        r = T.evaluate_continuous(ring, T.baseline(ring, "ring", "AR", 1, nb), "AR", 1, nb)["T_ns"]
        d = T.evaluate_continuous(ring, T.baseline(ring, "direct", "AR", 1, nb), "AR", 1, nb)["T_ns"]
        assert round(d / r, 2) == 12.88
        fc = T.Topology.from_workload_topology(W.fully_connected(100))
        r = T.evaluate_continuous(fc, T.baseline(fc, "ring", "AR", 1, nb), "AR", 1, nb)["T_ns"]
        d = T.evaluate_continuous(fc, T.baseline(fc, "direct", "AR", 1, nb), "AR", 1, nb)["T_ns"]
        assert round(r / d, 2) == 99.00


def test_greedy_beats_baselines_on_mesh(T):
    """on the 10 x 10 mesh the topology-aware synthesized
    All-Reduce is faster than both Ring and Direct (the paper reports 3.94x and
    5.52x; the ordering is asserted, the ratio recorded)."""
    topo = W.mesh2d(10, 10)
    t = T.Topology.from_workload_topology(topo)
    syn = oracle.synthesize(topo, 1, MiB, "AR", list(range(4)))
    g = T.evaluate_continuous(t, syn.sends, "AR", 1, MiB)["T_ns"]
    r = T.evaluate_continuous(t, T.baseline(t, "ring", "AR", 1, MiB), "AR", 1, MiB)["T_ns"]
    d = T.evaluate_continuous(t, T.baseline(t, "direct", "AR", 1, MiB), "AR", 1, MiB)["T_ns"]
    assert g < r < d
    assert r / g > 2 and d / g > 5


def test_closed_forms(T):
    """Single send: alpha + n / bw; two sends on one link serialize;
    uni ring All-Gather (Ring baseline and TACOS schedule): (p - 1)(alpha + n/bw)
    per chunk round (north_star closed form)."""
    t = T.Topology(2, [0, 1], [1, 0], [500, 500], [100, 100])
    one = np.zeros(1, dtype=T.SEND_DTYPE)
    one[0] = (0, 0, 1, 0, 0, 10986)
    assert T.evaluate_continuous(t, one, "AG", 1, MiB)["T_ns"] == pytest.approx(500 + MiB / 100)
    two = np.zeros(2, dtype=T.SEND_DTYPE)
    two[0] = (0, 0, 1, 0, 0, 10986)
    two[1] = (1, 0, 1, 0, 0, 10986)
    pre = oracle.bits_from_sets(2, 2, {0: [0, 1]})
    post = oracle.bits_from_sets(2, 2, {0: [0, 1], 1: [0, 1]})
    rep = T.evaluate_continuous(t, two, "CUSTOM", 1, MiB, pre=pre, post=post, n_chunks=2)
    assert rep["T_ns"] == pytest.approx(2 * (500 + MiB / 100))
    for p in (3, 4, 8):
        topo = W.uni_ring(p)
        tt = T.Topology.from_workload_topology(topo)
        per = 500 + MiB / 100
        assert T.evaluate_continuous(tt, T.baseline(tt, "ring", "AG", 1, MiB), "AG", 1, MiB)["T_ns"] == pytest.approx(
            (p - 1) * per)
        syn = oracle.synthesize(topo, 1, MiB, "AR", [0])
        rep = T.evaluate_continuous(tt, syn.sends, "AR", 1, MiB)
        assert rep["T_ns"] == pytest.approx(2 * (p - 1) * per)
        assert rep["T_rs_ns"] == pytest.approx((p - 1) * per)


@pytest.mark.parametrize("name", ["uni5", "torus34", "mesh33_hetero", "rand8", "hybrid"])
@pytest.mark.parametrize("coll", ["AG", "RS", "AR"])
def test_baselines_and_evaluator_match_reference(T, name, coll):
    topo = {"uni5": W.uni_ring(5), "torus34": W.torus([3, 4]), "mesh33_hetero": W.mesh2d(3, 3, 200, 100),
            "rand8": W.random_strongly_connected(8, 20, 4, bws=(25, 50, 100), alphas=(0, 500)),
            "hybrid": W.remove_undirected_links(W.switch_hypercube_hybrid(4, 4, 20, 25), 0.05, 3)[0]}[name]
    t = T.Topology.from_workload_topology(topo)
    for alg in ("ring", "direct"):
        a = T.baseline(t, alg, coll, 2, 256 << 10)
        b = OE.baseline(topo, alg, coll, 2, 256 << 10)
        assert a.tobytes() == b.tobytes()
        rep = T.evaluate_continuous(t, a, coll, 2, 256 << 10)
        ref_T, ref_rs = OE.evaluate(topo, b, coll, 2, 256 << 10)
        assert rep["T_ns"] == pytest.approx(float(ref_T), rel=1e-12)
        assert rep["T_rs_ns"] == pytest.approx(float(ref_rs), rel=1e-12)
    syn = oracle.synthesize(topo, 2, 256 << 10, coll, [0, 1])
    rep = T.evaluate_continuous(t, syn.sends, coll, 2, 256 << 10)
    ref_T, _ = OE.evaluate(topo, syn.sends, coll, 2, 256 << 10)
    assert rep["T_ns"] == pytest.approx(float(ref_T), rel=1e-12)
    # discretization never under-estimates (ceiling per link): continuous <= discrete * f
    assert rep["T_ns"] <= syn.T + 1e-6


def test_evaluator_rejects_invalid(T):
    t = T.Topology.from_workload_topology(W.uni_ring(3))
    bad = np.zeros(1, dtype=T.SEND_DTYPE)
    bad[0] = (1, 0, 1, 0, 0, 10986)  # NPU 0 does not hold chunk 1
    with pytest.raises(T.TacosError) as e:
        T.evaluate_continuous(t, bad, "AG", 1, MiB)
    assert e.value.code == T.TACOS_E_VERIFY


def test_oracle_evaluator_pinned_to_paper_ratios():
    """oracle/evaluate.py on its own (no library): the paper's printed ratios
    P:L107 + P:L120 (100 NPUs, alpha = 0.5 us, 100 GB/s, All-Reduce): Direct is
    12.88x slower than Ring on the 100-NPU (bidirectional) ring, Ring 99x slower
    than Direct on FullyConnected(100) -- exact rational times, rounded as printed."""
    ring = W.bi_ring(100)
    r = OE.evaluate(ring, OE.baseline(ring, "ring", "AR", 1, MiB), "AR", 1, MiB)[0]
    d = OE.evaluate(ring, OE.baseline(ring, "direct", "AR", 1, MiB), "AR", 1, MiB)[0]
    assert round(float(d / r), 2) == 12.88
    fc = W.fully_connected(100)
    r = OE.evaluate(fc, OE.baseline(fc, "ring", "AR", 1, MiB), "AR", 1, MiB)[0]
    d = OE.evaluate(fc, OE.baseline(fc, "direct", "AR", 1, MiB), "AR", 1, MiB)[0]
    assert round(float(r / d), 2) == 99.00


def test_oracle_evaluator_closed_forms():
    """oracle/evaluate.py against closed forms written from P:L104 (a send lasts
    alpha + n / bw): one send; k sends of one link serialize (k (alpha + n/bw));
    the Ring baseline on a uni ring of p NPUs: AG (p - 1)(alpha + n/bw), AR twice
    that with the RS phase ending half way (textbook ring)."""
    from fractions import Fraction

    per = Fraction(500) + Fraction(MiB, 100)
    two = W.Topology(2, np.array([0, 1], np.int32), np.array([1, 0], np.int32), np.array([500, 500], np.uint32),
                     np.array([100, 100], np.uint32))
    one = np.zeros(1, dtype=oracle.SEND_DTYPE)
    one[0] = (1, 1, 0, 1, 0, 10986)
    assert OE.evaluate(two, one, "AG", 1, MiB) == (per, 0)
    for k in (2, 5):
        s = np.zeros(k, dtype=oracle.SEND_DTYPE)
        for j in range(k):
            s[j] = (j, 0, 1, 0, 0, 10986)
        assert OE.evaluate(two, s, "AG", k, MiB)[0] == k * per
    for p in (3, 4, 7):
        topo = W.uni_ring(p)
        assert OE.evaluate(topo, OE.baseline(topo, "ring", "AG", 1, MiB), "AG", 1, MiB)[0] == (p - 1) * per
        T_ar, T_rs = OE.evaluate(topo, OE.baseline(topo, "ring", "AR", 1, MiB), "AR", 1, MiB)
        assert (T_ar, T_rs) == (2 * (p - 1) * per, (p - 1) * per)
