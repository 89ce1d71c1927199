"""Pins of the CPU oracle against what the paper and mathematics fix
(SURVEY.md §8(c) P1-P12).  None of these re-types the oracle's formulas: each
expected value is a hand-worked example, a closed form, an independent
implementation (cuRAND's host Philox, an exhaustive optimum, a separate
schedule replay) or an invariant.  CPU only.
"""
import ctypes
import os

import numpy as np
import pytest

import oracle
import workloads as W
from bruteforce import allgather_masks, optimum
from verify import ag_sets, check, clean

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def run_ag(topo, k, nbytes, seed=0, f=1):
    w = oracle.link_costs(topo, nbytes, f)
    return oracle.greedy(topo.n_npus, topo.src, topo.dst, w, topo.n_npus * k, k, seed), w


# --------------------------------------------------------------------------
# P1: Philox4x32-10 (R2)
# --------------------------------------------------------------------------
def test_philox_known_answers():
    """Random123 known-answer vectors for philox4x32_10 (Salmon et al. SC'11),
    tests/golden/philox4x32_10_kat.txt."""
    n = 0
    with open(os.path.join(GOLDEN, "philox4x32_10_kat.txt")) as fh:
        for line in fh:
            if not line.strip() or line.startswith("#"):
                continue
            vals = [int(x, 16) for x in line.split()]
            ctr, key, out = vals[0:4], vals[4:6], vals[6:10]
            assert oracle.philox(ctr, key) == out
            n += 1
    assert n == 3


def _curand():
    for name in ("libcurand.so.10", "/usr/local/cuda/lib64/libcurand.so.10", "libcurand.so"):
        try:
            return ctypes.CDLL(name)
        except OSError:
            continue
    return None


@pytest.mark.parametrize("seed", [0, 1, 0x0123456789ABCDEF, 2**64 - 1])
def test_philox_matches_curand_host_generator(seed):
    """cuRAND's host PHILOX4_32_10 generator (an independent implementation)
    emits block i = Philox(ctr=(0,0,i,0), key=seed) -- exactly the oracle's
    draw counter for time 0, link i, sigma 0."""
    cr = _curand()
    if cr is None:
        pytest.skip("libcurand not available")
    g = ctypes.c_void_p()
    assert cr.curandCreateGeneratorHost(ctypes.byref(g), 161) == 0  # CURAND_RNG_PSEUDO_PHILOX4_32_10
    try:
        assert cr.curandSetPseudoRandomGeneratorSeed(g, ctypes.c_ulonglong(seed)) == 0
        n_blocks = 64
        out = np.zeros(4 * n_blocks, np.uint32)
        assert cr.curandGenerate(g, out.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(out.size)) == 0
    finally:
        cr.curandDestroyGenerator(g)
    key = [seed & 0xFFFFFFFF, seed >> 32]
    for i in range(n_blocks):
        assert oracle.philox([0, 0, i, 0], key) == out[4 * i: 4 * i + 4].tolist()


def _curand_blocks(seed, n_blocks):
    cr = _curand()
    if cr is None:
        pytest.skip("libcurand not available")
    g = ctypes.c_void_p()
    assert cr.curandCreateGeneratorHost(ctypes.byref(g), 161) == 0
    cr.curandSetPseudoRandomGeneratorSeed(g, ctypes.c_ulonglong(seed))
    out = np.zeros(4 * n_blocks, np.uint32)
    cr.curandGenerate(g, out.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(out.size))
    cr.curandDestroyGenerator(g)
    return out.reshape(n_blocks, 4)


@pytest.mark.parametrize("seed", list(range(12)))
def test_first_event_draws_follow_curand_stream(seed):
    """Two equal-cost in-links 0->2 (link 0) and 1->2 (link 1); NPUs 0 and 1 both
    hold chunks {0,1}, NPU 2 needs both.  At t=0 the links are walked in
    ascending u_ord = word0 (R3), the first one picks the r-th candidate with
    r = floor(word1 * 2 / 2^32) (R13), the second gets the other chunk.  The
    expected outcome is computed from cuRAND's stream, not from the oracle."""
    blocks = _curand_blocks(seed, 2)
    pre = oracle.bits_from_sets(3, 2, {0: [0, 1], 1: [0, 1]})
    post = oracle.bits_from_sets(3, 2, {0: [0, 1], 1: [0, 1], 2: [0, 1]})
    src = np.array([0, 1], np.int32)
    dst = np.array([2, 2], np.int32)
    w = np.array([5, 5], np.uint64)
    res = oracle.greedy(3, src, dst, w, 2, 1, seed, 0, pre, post)
    first = 0 if int(blocks[0, 0]) < int(blocks[1, 0]) else 1
    r = (int(blocks[first, 1]) * 2) >> 32
    got = {int(s["link"]): int(s["chunk"]) for s in res.sends}
    assert got[first] == r
    assert got[1 - first] == 1 - r
    assert res.T == 5


@pytest.mark.parametrize("seed", [3, 0xFEEDFACE, 2**63 + 5])
def test_first_event_select_across_words_follows_curand_stream(seed):
    """Cross-word rank-select (R12, R13): a star, link i = 0 -> i+1 (i < 24), one
    in-link per destination.  NPU 0 holds a random set S of the C = 160 chunks
    (5 words), NPU i+1 a random set H_i.  At t = 0 link i takes the r-th smallest
    member of S - H_i with r = floor(word1 * K / 2^32), K = |S - H_i|, word1 of
    cuRAND's block i (counter (0, 0, i, 0)).  The expected chunk is computed from
    cuRAND's stream and a sorted Python list, not from the oracle; the candidate
    sets span every word, so a slip in the word walk changes the outcome."""
    n_links, C = 24, 160
    rng = np.random.default_rng(seed % 2**32)
    S = sorted(set(rng.choice(C, 90, replace=False).tolist()))
    H = [set(rng.choice(C, int(rng.integers(0, 60)), replace=False).tolist()) for _ in range(n_links)]
    blocks = _curand_blocks(seed, n_links)
    pre_sets = {0: S}
    post_sets = {0: S}
    for i in range(n_links):
        pre_sets[i + 1] = sorted(H[i])
        post_sets[i + 1] = sorted(set(S) | H[i])
    n = n_links + 1
    pre = oracle.bits_from_sets(n, C, pre_sets)
    post = oracle.bits_from_sets(n, C, post_sets)
    src = np.zeros(n_links, np.int32)
    dst = np.arange(1, n, dtype=np.int32)
    w = np.full(n_links, 7, np.uint64)
    res = oracle.greedy(n, src, dst, w, C, 1, seed, 0, pre, post)
    first = {int(e["link"]): int(e["chunk"]) for e in res.sends if int(e["t_start"]) == 0}
    words_hit = set()
    for i in range(n_links):
        cand = [c for c in S if c not in H[i]]
        r = (int(blocks[i, 1]) * len(cand)) >> 32
        assert first[i] == cand[r], (i, first[i], cand[r])
        words_hit.add(cand[r] >> 5)
    assert words_hit == set(range(C // 32))  # the picks land in every word


# --------------------------------------------------------------------------
# a1 cost quantization (R5, R6)
# --------------------------------------------------------------------------
def test_link_cost_hand_values():
    # 1 MiB at 100 B/ns: 1,048,576/100 = 10,485.76 -> 10,486; + 500 ns alpha
    assert oracle.link_cost(500, 100, 1 << 20) == 10986
    # 128 KiB at 200 / 100 B/ns: 655.36 -> 656 ; 1310.72 -> 1311
    assert oracle.link_cost(500, 200, 128 << 10) == 1156
    assert oracle.link_cost(500, 100, 128 << 10) == 1811
    # 1 MiB at 20 / 25 B/ns: 52,428.8 -> 52,429 ; 41,943.04 -> 41,944
    assert oracle.link_cost(500, 20, 1 << 20) == 52929
    assert oracle.link_cost(500, 25, 1 << 20) == 42444
    # exact multiples are not rounded up; the ceiling is per link
    assert oracle.link_cost(0, 4, 40) == 10
    assert oracle.link_cost(0, 4, 41) == 11
    assert oracle.link_cost(10, 1, 0) == 10
    # discretization factor f (P:L172 ceil(l/f)): l = 10 ns -> f=3: ceil(3.33) = 4
    assert oracle.link_cost(10, 1, 0, 3) == 4
    assert oracle.link_cost(9, 1, 0, 3) == 3
    # l = 500 + 10485.76 = 10985.76 ns; f = 1000 -> 11 steps; f = 10986 -> 1
    assert oracle.link_cost(500, 100, 1 << 20, 1000) == 11
    assert oracle.link_cost(500, 100, 1 << 20, 10986) == 1
    assert oracle.link_cost(500, 100, 1 << 20, 10985) == 2
    # large values: alpha*bw overflows 32 bits but the result is exact
    assert oracle.link_cost(4_000_000_000, 4_000_000_000, 0, 4_000_000_000) == 1
    assert oracle.link_cost(1, 3_000_000_000, 2**40, 1) == 1 + (2**40 + 3_000_000_000 - 1) // 3_000_000_000


def test_link_cost_errors():
    with pytest.raises(oracle.OracleError):
        oracle.link_cost(500, 0, 1)  # bw = 0
    with pytest.raises(oracle.OracleError):
        oracle.link_cost(0, 7, 0)  # zero delay: w would be 0
    with pytest.raises(oracle.OracleError):
        oracle.link_cost(4_000_000_000, 1, 2**62, 1)  # > 2^32 time units


# --------------------------------------------------------------------------
# P2 uni ring: T = (p-1) w, unique schedule; config 1 exactly
# --------------------------------------------------------------------------
def test_config1_exact_schedule():
    """SURVEY P2 hand-worked: 4-NPU uni ring, w = 10,986, T = 32,958, 12 sends.
    tests/golden/config1_ag.txt."""
    wl = W.config(1)
    want = []
    with open(os.path.join(GOLDEN, "config1_ag.txt")) as fh:
        for line in fh:
            if line.strip() and not line.startswith("#"):
                want.append(tuple(int(x) for x in line.split()))
    for seed in range(17):
        syn = oracle.synthesize(wl.topo, 1, wl.chunk_bytes, "AG", [seed])
        assert syn.T == 32958
        got = [tuple(int(r[f]) for f in ("chunk", "src", "dst", "link", "t_start", "t_end")) for r in syn.sends]
        assert got == want


@pytest.mark.parametrize("p", [2, 3, 4, 5, 7, 9])
@pytest.mark.parametrize("k", [1, 2, 3])
def test_uni_ring_closed_form(p, k):
    """Ring All-Gather closed form (p-1)(alpha + n/beta) (north_star; SPEC
    S:L435) for k = 1.  With k > 1 chunks per NPU the single in-link must
    carry (p-1)k chunks, so T >= (p-1) k w; the random pick may
    forward a relayed chunk early and leave the link idle later, so only the
    bound is fixed."""
    topo = W.uni_ring(p, 100)
    for seed in range(5):
        res, w = run_ag(topo, k, 1 << 20, seed)
        if k == 1:
            assert res.T == (p - 1) * int(w[0])
        else:
            assert res.T >= (p - 1) * k * int(w[0])
            assert res.T % int(w[0]) == 0
        rep = check(p, topo.src, topo.dst, w, res.sends, *ag_sets(p, k))
        assert clean(rep), rep
        if k == 1:  # unique schedule: link i at step j carries chunk (i - j) mod p
            for s in res.sends:
                j = int(s["t_start"]) // int(w[0])
                assert int(s["chunk"]) == (int(s["src"]) - j) % p


@pytest.mark.parametrize("p", [3, 4, 5, 6, 8, 11])
def test_bi_ring_closed_form(p):
    """bidirectional ring, k=1: T = ceil((p-1)/2) w for every seed."""
    topo = W.bi_ring(p, 100)
    for seed in range(8):
        res, w = run_ag(topo, 1, 1 << 20, seed)
        assert res.T == ((p - 1 + 1) // 2) * int(w[0])
        assert clean(check(p, topo.src, topo.dst, w, res.sends, *ag_sets(p, 1)))


@pytest.mark.parametrize("p", [2, 3, 5, 8])
def test_path_closed_form(p):
    """path (1-D mesh), k=1: T = (p-1) w."""
    topo = W.path(p, 100)
    for seed in range(4):
        res, w = run_ag(topo, 1, 1 << 20, seed)
        assert res.T == (p - 1) * int(w[0])


@pytest.mark.parametrize("n", [2, 3, 5, 8])
def test_fully_connected_one_step(n):
    """FC(n), k=1: every NPU receives every chunk directly at t=0."""
    topo = W.fully_connected(n, 100)
    res, w = run_ag(topo, 1, 1 << 20, 3)
    assert res.T == int(w[0])
    assert len(res.sends) == n * (n - 1)
    assert all(int(s["t_start"]) == 0 and int(s["chunk"]) == int(s["src"]) for s in res.sends)


def test_mesh2x2_diagonal_split():
    """2x2 mesh (a bidirectional 4-ring): T = 2w; at step 2 exactly
    one of each node's two in-links carries the diagonal chunk, which one
    depends on the seed (both outcomes occur; the Philox order key decides)."""
    topo = W.mesh2d(2, 2)
    counts = {}
    for seed in range(200):
        res, w = run_ag(topo, 1, 1 << 20, seed)
        assert res.T == 2 * int(w[0])
        step2 = [s for s in res.sends if int(s["t_start"]) == int(w[0])]
        assert len(step2) == 4
        diag = {0: 3, 1: 2, 2: 1, 3: 0}
        for s in step2:
            assert int(s["chunk"]) == diag[int(s["dst"])]
        key = tuple(sorted(int(s["link"]) for s in step2))
        counts[key] = counts.get(key, 0) + 1
    # 4 destinations x 2 choices each, independent: 16 patterns, all seen
    assert len(counts) == 16
    assert max(counts.values()) < 40


# --------------------------------------------------------------------------
# P7 heterogeneous hand examples (Fig. HeterogeneousGreedy)
# --------------------------------------------------------------------------
def _custom(n, links, C, pre, post, seeds=range(16)):
    src = np.array([l[0] for l in links], np.int32)
    dst = np.array([l[1] for l in links], np.int32)
    w = np.array([l[2] for l in links], np.uint64)
    preb = oracle.bits_from_sets(n, C, pre)
    postb = oracle.bits_from_sets(n, C, post)
    outs = []
    for s in seeds:
        r = oracle.greedy(n, src, dst, w, C, 1, s, 0, preb, postb)
        outs.append(r)
    return outs


def _tuples(r):
    return sorted((int(s["chunk"]), int(s["src"]), int(s["dst"]), int(s["t_start"]), int(s["t_end"])) for s in r.sends)


def test_E5_shorter_link_first():
    """Fig. HeterogeneousGreedy(a): two in-links to NPU 2, link ids
    in the opposite order of their costs: l0 = 1->2 (w=2), l1 = 0->2 (w=1)."""
    for r in _custom(3, [(1, 2, 2), (0, 2, 1)], 1, {0: [0], 1: [0]}, {0: [0], 1: [0], 2: [0]}):
        assert _tuples(r) == [(0, 0, 2, 0, 1)]
        assert r.T == 1


def test_E6_arrival_time():
    """Fig. HeterogeneousGreedy(b): chunk on NPU 2 reaches 1 at t=2
    over a 2-step link; 1 cannot forward it at t=1."""
    for r in _custom(3, [(2, 1, 2), (1, 0, 1)], 1, {2: [0]}, {0: [0], 1: [0], 2: [0]}):
        assert _tuples(r) == [(0, 1, 0, 2, 3), (0, 2, 1, 0, 2)]
        assert r.T == 3


def test_E7_persistent_claim():
    """R4 (contrast Fig. HeterogeneousGreedy(c)): c0 claimed for
    NPU 2 over the 3-step link at t=0 is withheld from 1->2 at t=1."""
    for r in _custom(3, [(0, 2, 3), (0, 1, 1), (1, 2, 1)], 1, {0: [0]}, {0: [0], 1: [0], 2: [0]}):
        assert _tuples(r) == [(0, 0, 1, 0, 1), (0, 0, 2, 0, 3)]
        assert r.T == 3
    # the exhaustive optimum relays through NPU 1 and finishes at 2 (P10)
    assert optimum(3, [(0, 2, 3), (0, 1, 1), (1, 2, 1)], [1, 0, 0], [1, 1, 1]) == 2


def test_custom_stall_is_unreachable():
    """R17: a CUSTOM postcondition needing a relay through an NPU that does not
    request the chunk stalls; the oracle reports UNREACHABLE."""
    with pytest.raises(oracle.OracleError) as e:
        _custom(3, [(0, 1, 1), (1, 2, 1)], 1, {0: [0]}, {0: [0], 2: [0]}, seeds=[0])
    assert e.value.code == oracle.E_UNREACHABLE


# --------------------------------------------------------------------------
# P8 uni ring All-Reduce; P12 inversion
# --------------------------------------------------------------------------
@pytest.mark.parametrize("p", [3, 4, 6])
def test_uni_ring_allreduce(p):
    """P:L91 AR = RS then AG; RS of the (asymmetric) uni ring = mirror of the
    AG on the reversed ring (R9).  Textbook ring: T_AR = 2 (p-1) w."""
    topo = W.uni_ring(p, 100)
    syn = oracle.synthesize(topo, 1, 1 << 20, "AR", list(range(4)))
    w = int(oracle.link_cost(500, 100, 1 << 20))
    assert syn.T == 2 * (p - 1) * w
    assert syn.T_rs == syn.T_ag == (p - 1) * w
    assert len(syn.sends) == 2 * p * (p - 1)
    # every AR send uses a real link of G (the uni ring), never a reverse link
    for s in syn.sends:
        assert int(topo.dst[int(s["link"])]) == int(s["dst"]) and int(topo.src[int(s["link"])]) == int(s["src"])


@pytest.mark.parametrize("cfg_topo", ["torus44", "uni5", "rand"])
def test_inversion_properties(cfg_topo):
    """P12: mirror o mirror = id; horizon and send count preserved; the RS half
    mirrored back verifies as an All-Gather on G^T; T_AR = T_RS + T_AG; the RS
    half ends exactly where the AG half begins."""
    topo = {"torus44": W.torus([4, 4]), "uni5": W.uni_ring(5), "rand": W.random_strongly_connected(6, 14, 3)}[cfg_topo]
    k = 2
    syn = oracle.synthesize(topo, k, 1 << 20, "AR", [0, 1, 2])
    w = oracle.link_costs(topo, 1 << 20)
    rs = syn.sends[syn.sends["t_end"] <= syn.T_rs]
    ag = syn.sends[syn.sends["t_start"] >= syn.T_rs]
    assert len(rs) + len(ag) == len(syn.sends) == 2 * topo.n_npus * k * (topo.n_npus - 1)
    assert syn.T == syn.T_rs + syn.T_ag
    # RS back to AG on G^T: (c, b->a, T-t1, T-t0) lands on link id j of G^T
    back = oracle.mirror(rs, syn.T_rs, topo.src, topo.dst, None)
    gt = W.transpose(topo)
    rep = check(topo.n_npus, gt.src, gt.dst, w, back, *ag_sets(topo.n_npus, k), greedy=False)
    assert clean(rep), rep
    assert rep["T"] == syn.T_rs
    twice = oracle.mirror(back, syn.T_rs, gt.src, gt.dst, None)
    assert np.array_equal(oracle.canonical(twice), oracle.canonical(rs))
    ag0 = ag.copy()
    ag0["t_start"] -= np.uint64(syn.T_rs)
    ag0["t_end"] -= np.uint64(syn.T_rs)
    rep2 = check(topo.n_npus, topo.src, topo.dst, w, ag0, *ag_sets(topo.n_npus, k))
    assert clean(rep2), rep2


# --------------------------------------------------------------------------
# P9 lower bounds; P11 invariants; determinism; best-of-S
# --------------------------------------------------------------------------
def _per_node_bound(topo, w, k):
    """smallest T with sum over in-links of floor(T/w) >= C - k, max over nodes"""
    C = topo.n_npus * k
    ins = [[] for _ in range(topo.n_npus)]
    for l in range(topo.n_links):
        ins[int(topo.dst[l])].append(int(w[l]))
    best = 0
    for ws in ins:
        lo, hi = 0, (C - k) * max(ws)  # sum(floor(T/w)) is monotone in T: bisect
        while lo < hi:
            mid = (lo + hi) // 2
            if sum(mid // q for q in ws) >= C - k:
                hi = mid
            else:
                lo = mid + 1
        best = max(best, lo)
    return best


def test_mesh3x3_bound_from_paper_example():
    """P:L333 (Fig. MeshExampleSearchResult, 3x3 mesh AG): a corner has in-degree
    2 and needs 8 chunks, so T_AG >= 4 w for every seed."""
    topo = W.mesh2d(3, 3)
    for seed in range(10):
        res, w = run_ag(topo, 1, 1 << 20, seed)
        assert res.T >= 4 * int(w[0])
        assert clean(check(9, topo.src, topo.dst, w, res.sends, *ag_sets(9, 1)))


@pytest.mark.parametrize("i", [2, 3])
def test_config_lower_bounds(i):
    """config 2 T_AG >= 63 w = 692,118; config 3 T_AG >= 86 w = 944,796
    (per-node in-link bound; config 3 also diameter 12)."""
    wl = W.config(i)
    syn = oracle.synthesize(wl.topo, wl.chunks_per_npu, wl.chunk_bytes, "AR", list(range(4)))
    bound = {2: 692118, 3: 944796}[i]
    for g in syn.ag:
        assert g.T >= bound
        assert g.M == wl.topo.n_npus * wl.chunks_per_npu * (wl.topo.n_npus - 1)
    w = oracle.link_costs(wl.topo, wl.chunk_bytes)
    assert _per_node_bound(wl.topo, w, wl.chunks_per_npu) == bound
    assert syn.T == 2 * min(g.T for g in syn.ag)


@pytest.mark.parametrize("name", ["torus44", "mesh34_hetero", "hypercube3", "rand7", "hybrid"])
def test_invariants_every_seed(name):
    """SURVEY P11 on every produced schedule: exactly-once delivery, held at
    departure, durations, disjoint link intervals, T = max t_end, maximality
    and shorter-link-first at every event."""
    topo = {
        "torus44": W.torus([4, 4]),
        "mesh34_hetero": W.mesh2d(3, 4, 200, 100),
        "hypercube3": W.hypercube(3, 50),
        "rand7": W.random_strongly_connected(7, 20, 11, bws=(25, 50, 100), alphas=(0, 500, 1500)),
        "hybrid": W.remove_undirected_links(W.switch_hypercube_hybrid(4, 4, 20, 25), 0.05, 1)[0],
    }[name]
    k = 2
    for seed in range(6):
        res, w = run_ag(topo, k, 256 << 10, seed)
        rep = check(topo.n_npus, topo.src, topo.dst, w, res.sends, *ag_sets(topo.n_npus, k))
        assert clean(rep), (seed, {a: b[:5] for a, b in rep.items() if a != "T"})
        assert rep["T"] == res.T
        assert res.M == len(res.sends) == topo.n_npus * k * (topo.n_npus - 1)
        assert _per_node_bound(topo, w, k) <= res.T


def test_determinism_and_best_of_s():
    """Three runs byte-identical; best-of-S T is non-increasing in S
     and equals the minimum over single-seed runs."""
    wl = W.config(2)
    runs = [oracle.synthesize(wl.topo, wl.chunks_per_npu, wl.chunk_bytes, "AR", list(range(6))) for _ in range(3)]
    for r in runs[1:]:
        assert r.T == runs[0].T and r.sends.tobytes() == runs[0].sends.tobytes()
    prev = None
    singles = [oracle.synthesize(wl.topo, wl.chunks_per_npu, wl.chunk_bytes, "AR", [s]).T for s in range(8)]
    for S in range(1, 9):
        T = oracle.synthesize(wl.topo, wl.chunks_per_npu, wl.chunk_bytes, "AR", list(range(S))).T
        assert T == min(singles[:S])
        if prev is not None:
            assert T <= prev
        prev = T


# --------------------------------------------------------------------------
# P10 brute force on tiny instances
# --------------------------------------------------------------------------
@pytest.mark.parametrize("inst", range(14))
def test_greedy_never_beats_exhaustive_optimum(inst):
    """SURVEY P10 (SPEC S:L316, S:L619 adapted): random strongly connected
    digraphs, <= 4 NPUs, <= 6 links, <= 4 chunks, w in {1,2,3}: the greedy
    finishing time is >= the exhaustive optimum, for every seed.  On
    instances with unit costs and one chunk per NPU the greedy is optimal
    often; the rate is recorded, not asserted."""
    rng = np.random.default_rng(1000 + inst)
    n = int(rng.integers(2, 5))
    L = int(rng.integers(n, min(6, n * (n - 1)) + 1))
    topo = W.random_strongly_connected(n, L, 1000 + inst)
    k = 1 if n > 2 else int(rng.integers(1, 3))
    w = rng.integers(1, 4, size=topo.n_links).astype(np.uint64)
    links = [(int(s), int(d), int(x)) for s, d, x in zip(topo.src, topo.dst, w)]
    pre, post = allgather_masks(n, k)
    t_opt = optimum(n, links, pre, post)
    assert t_opt is not None
    for seed in range(8):
        r = oracle.greedy(n, topo.src, topo.dst, w, n * k, k, seed)
        assert r.T >= t_opt
        assert clean(check(n, topo.src, topo.dst, w, r.sends, *ag_sets(n, k)))


def test_bruteforce_self_check():
    """The exhaustive search itself on closed forms: uni ring 4 (w=1): 3;
    FC(3): 1; path 3 with w=2: 4; 2-NPU, k=2, w=1: 2."""
    assert optimum(4, [(i, (i + 1) % 4, 1) for i in range(4)], *allgather_masks(4, 1)) == 3
    assert optimum(3, [(a, b, 1) for a in range(3) for b in range(3) if a != b], *allgather_masks(3, 1)) == 1
    assert optimum(3, [(0, 1, 2), (1, 0, 2), (1, 2, 2), (2, 1, 2)], *allgather_masks(3, 1)) == 4
    assert optimum(2, [(0, 1, 1), (1, 0, 1)], *allgather_masks(2, 2)) == 2


# --------------------------------------------------------------------------
# Paper-literal variant (row f1, reading R21): chunk-first + replacement
# --------------------------------------------------------------------------
def _custom_literal(n, links, C, pre, post, seeds=range(16)):
    src = np.array([l[0] for l in links], np.int32)
    dst = np.array([l[1] for l in links], np.int32)
    w = np.array([l[2] for l in links], np.uint64)
    preb = oracle.bits_from_sets(n, C, pre)
    postb = oracle.bits_from_sets(n, C, post)
    return [oracle.greedy(n, src, dst, w, C, 1, s, 0, preb, postb, literal=True) for s in seeds]


def test_literal_replacement_fig_heterogeneous_c():
    """Fig. HeterogeneousGreedy(c): the chunk requested at t=0 over the
    slow link 0->2 (w=3) is requested again at t=1 over 1->2 once NPU 1 holds it;
    it arrives at t=2 and the copy still on 0->2 is outdated and cancelled.
    Every seed: T = 2, sends {(c0, 0->1, 0, 1), (c0, 1->2, 1, 2)}, one cancellation.
    (Link-first with persistent claims gives T = 3 on the same instance, E7.)"""
    for r in _custom_literal(3, [(0, 2, 3), (0, 1, 1), (1, 2, 1)], 1, {0: [0]}, {0: [0], 1: [0], 2: [0]}):
        assert _tuples(r) == [(0, 0, 1, 0, 1), (0, 1, 2, 1, 2)]
        assert r.T == 2 and r.X == 1 and r.M == 3


def test_literal_shorter_first_and_arrival_time():
    """E5 and E6 hold for the literal variant too."""
    for r in _custom_literal(3, [(1, 2, 2), (0, 2, 1)], 1, {0: [0], 1: [0]}, {0: [0], 1: [0], 2: [0]}):
        assert _tuples(r) == [(0, 0, 2, 0, 1)] and r.T == 1
    for r in _custom_literal(3, [(2, 1, 2), (1, 0, 1)], 1, {2: [0]}, {0: [0], 1: [0], 2: [0]}):
        assert _tuples(r) == [(0, 1, 0, 2, 3), (0, 2, 1, 0, 2)] and r.T == 3


@pytest.mark.parametrize("p", [3, 4, 7])
def test_literal_closed_forms(p):
    """Uni ring (p-1)w, bi ring ceil((p-1)/2)w, FC w: unique frontiers, so the
    literal variant matches the closed forms (and never cancels)."""
    for topo, want in ((W.uni_ring(p), (p - 1)), (W.bi_ring(p), (p - 1 + 1) // 2), (W.fully_connected(p), 1)):
        w = oracle.link_costs(topo, 1 << 20)
        for seed in range(4):
            r = oracle.greedy(p, topo.src, topo.dst, w, p, 1, seed, literal=True)
            assert r.T == want * int(w[0]) and r.X == 0


@pytest.mark.parametrize("name", ["torus44", "mesh34_hetero", "rand7", "hybrid"])
def test_literal_invariants(name):
    """The final literal schedule is a valid congestion-free AG: exactly-once
    delivery, arrival before departure, durations, disjoint link intervals;
    issued = delivered + cancelled."""
    topo = {
        "torus44": W.torus([4, 4]),
        "mesh34_hetero": W.mesh2d(3, 4, 200, 100),
        "rand7": W.random_strongly_connected(7, 20, 11, bws=(25, 50, 100), alphas=(0, 500, 1500)),
        "hybrid": W.remove_undirected_links(W.switch_hypercube_hybrid(4, 4, 20, 25), 0.05, 1)[0],
    }[name]
    k = 2
    w = oracle.link_costs(topo, 256 << 10)
    for seed in range(6):
        r = oracle.greedy(topo.n_npus, topo.src, topo.dst, w, topo.n_npus * k, k, seed, literal=True)
        rep = check(topo.n_npus, topo.src, topo.dst, w, r.sends, *ag_sets(topo.n_npus, k), greedy=False)
        assert clean(rep), rep
        assert rep["T"] == r.T
        assert len(r.sends) == topo.n_npus * k * (topo.n_npus - 1) == r.M - r.X


@pytest.mark.parametrize("inst", range(8))
def test_literal_never_beats_exhaustive_optimum(inst):
    rng = np.random.default_rng(2000 + inst)
    n = int(rng.integers(2, 5))
    L = int(rng.integers(n, min(6, n * (n - 1)) + 1))
    topo = W.random_strongly_connected(n, L, 2000 + inst)
    w = rng.integers(1, 4, size=topo.n_links).astype(np.uint64)
    links = [(int(s), int(d), int(x)) for s, d, x in zip(topo.src, topo.dst, w)]
    t_opt = optimum(n, links, *allgather_masks(n, 1))
    for seed in range(8):
        r = oracle.greedy(n, topo.src, topo.dst, w, n, 1, seed, literal=True)
        assert r.T >= t_opt


def test_best_of_s_bookkeeping_r24():
    """Reading R24: per-seed collective times and searched jobs.  Symmetric graph: one search
    per seed, T_AR(s) = 2 T_AG(s).  Asymmetric graph: AR searches G and G^T per seed,
    T_AR(s) = T_RS(s) + T_AG(s), the winners are chosen independently (T_AR = min T_RS +
    min T_AG, P:L274 / R9 / R10); an RS alone searches only G^T."""
    seeds = [0, 1, 2, 3, 4]
    sym = oracle.synthesize(W.torus([3, 4]), 1, 1 << 20, "AR", seeds)
    assert sym.rs is sym.ag and len(sym.ag) == 5
    assert [int(x) for x in sym.seed_times] == [2 * g.T for g in sym.ag]
    topo = W.random_strongly_connected(8, 19, 4, bws=(25, 50, 100), alphas=(0, 500))
    ar = oracle.synthesize(topo, 2, 1 << 20, "AR", seeds)
    assert ar.rs is not ar.ag and len(ar.ag) == len(ar.rs) == 5
    assert all(g.sigma == 0 for g in ar.ag) and all(g.sigma == 1 for g in ar.rs)
    assert [int(x) for x in ar.seed_times] == [r.T + g.T for r, g in zip(ar.rs, ar.ag)]
    assert ar.T == min(r.T for r in ar.rs) + min(g.T for g in ar.ag)
    rs = oracle.synthesize(topo, 2, 1 << 20, "RS", seeds)
    assert rs.ag == [] and len(rs.rs) == 5 and all(r.sigma == 1 for r in rs.rs)
    assert [int(x) for x in rs.seed_times] == [r.T for r in ar.rs]
    assert rs.T == min(r.T for r in ar.rs)
