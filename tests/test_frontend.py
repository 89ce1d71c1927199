"""Topology front-end of the library: hierarchical
composition with switch unwinding (§IV.D) and NPU
removal, against the plain-loop reference in
oracle/topology.py, the input generators of workloads/, and the paper's
stated sizes.  CPU only (host code)."""
import numpy as np
import pytest

import oracle
import oracle.topology as OT
import workloads as W


@pytest.fixture(scope="module")
def T():
    from paper_2304_05301_b200 import build

    build.build()
    import paper_2304_05301_b200 as T

    T.load_library()
    return T


def as_list(n, src, dst, al, bw):
    return n, list(zip(src.tolist(), dst.tolist(), al.tolist(), bw.tolist()))


def test_switch_unwinding_paper_figure(T):
    """Fig. UnwindSwitch: a 4-NPU switch at 120 GB/s; degree d gives
    n -> n+1..n+d with 120/d GB/s each; d = 1 keeps the full 120 GB/s (and has a
    bi-directional ring variation); d = 3 on 4 NPUs is fully connected."""
    for d, per_link in ((1, 120), (2, 60), (3, 40)):
        n, links = as_list(*T.tacos_build_hierarchical([{"kind": "switch", "n": 4, "degree": d, "bw": 120}]))
        assert n == 4 and len(links) == 4 * d
        assert all(bw == per_link for *_, bw in links)
        assert sorted((a, b) for a, b, *_ in links) == sorted((i, (i + s) % 4) for i in range(4) for s in range(1, d + 1))
    n, links = as_list(*T.tacos_build_hierarchical([{"kind": "switch", "n": 4, "degree": 1, "bidirectional": 1,
                                                    "bw": 120}]))
    assert len(links) == 8 and all(bw == 120 for *_, bw in links)
    _, fc = as_list(*T.tacos_build_hierarchical([{"kind": "fc", "n": 4, "bw": 40}]))
    _, sw3 = as_list(*T.tacos_build_hierarchical([{"kind": "switch", "n": 4, "degree": 3, "bw": 120}]))
    assert sorted(fc) == sorted(sw3)


def test_products_equal_input_generators(T):
    """A 3-D torus is Ring x Ring x Ring (bi-directional) and a 2-D mesh is
    Path x Path: the front-end reproduces workloads' generators link for link
    (same canonical order)."""
    for dims, ref in (
        ([{"kind": "ring", "n": 8, "bidirectional": 1, "bw": 100}] * 3, W.torus([8, 8, 8], 100)),
        ([{"kind": "ring", "n": 5, "bidirectional": 1, "bw": 100}, {"kind": "ring", "n": 3, "bidirectional": 1, "bw": 100}],
         W.torus([5, 3], 100)),
        ([{"kind": "path", "n": 32, "bw": 200}, {"kind": "path", "n": 32, "bw": 100}], W.mesh2d(32, 32, 200, 100)),
    ):
        n, src, dst, al, bw = T.tacos_build_hierarchical(dims)
        assert n == ref.n_npus
        assert np.array_equal(src, ref.src) and np.array_equal(dst, ref.dst)
        assert np.array_equal(al, ref.alpha_ns) and np.array_equal(bw, ref.bw)


def test_paper_ring_fc_switch_512(T):
    """Ring_FC_Switch with node 2 x 4 and 64 nodes (512 NPUs), degree-1
    scale-out switch: N = 512, L = 512 * (1 + 3 + 1) = 2560 (SURVEY §8(d) ctx row);
    identical to workloads.ring_fc_switch; asymmetric; strongly connected."""
    dims = [{"kind": "ring", "n": 2, "bw": 200}, {"kind": "fc", "n": 4, "bw": 100},
            {"kind": "switch", "n": 64, "degree": 1, "bw": 50}]
    n, src, dst, al, bw = T.tacos_build_hierarchical(dims)
    assert (n, len(src)) == (512, 2560)
    ref = W.ring_fc_switch(2, 4, 64)
    assert np.array_equal(src, ref.src) and np.array_equal(dst, ref.dst) and np.array_equal(bw, ref.bw)
    t = T.Topology(n, src, dst, al, bw)
    assert t.strongly_connected and not t.is_symmetric(1 << 20)


@pytest.mark.parametrize("seed", range(8))
def test_random_products_match_reference(T, seed):
    rng = np.random.default_rng(seed)
    kinds = ["ring", "fc", "switch", "path"]
    dims = []
    for _ in range(int(rng.integers(1, 4))):
        k = kinds[int(rng.integers(0, 4))]
        n = int(rng.integers(2, 6))
        d = {"kind": k, "n": n, "alpha_ns": int(rng.integers(0, 1000)), "bidirectional": int(rng.integers(0, 2))}
        if k == "switch":
            d["degree"] = int(rng.integers(1, n))
            d["bw"] = d["degree"] * int(rng.integers(1, 50))
        else:
            d["bw"] = int(rng.integers(1, 400))
        dims.append(d)
    n, src, dst, al, bw = T.tacos_build_hierarchical(dims)
    n2, ref = OT.hierarchical(dims)
    assert n == n2
    assert list(zip(src.tolist(), dst.tolist(), al.tolist(), bw.tolist())) == ref


def test_npu_removal_table_iv(T):
    """Table IV: a 4 x 4 mesh without NPUs 7 and 9 keeps 14 NPUs;
    NPU 7 (x=3, y=1) has 3 neighbours and NPU 9 (x=1, y=2) 4, not adjacent:
    48 - 2*(3 + 4) = 34 directed links remain, still strongly connected."""
    m = W.mesh2d(4, 4)
    n2, src, dst, al, bw, old = T.tacos_remove_npus(16, m.src, m.dst, m.alpha_ns, m.bw, [7, 9])
    assert (n2, len(src)) == (14, 34)
    assert old.tolist() == [x for x in range(16) if x not in (7, 9)]
    n3, ref, keep = OT.remove_npus(16, m.links(), [7, 9])
    assert list(zip(src.tolist(), dst.tolist(), al.tolist(), bw.tolist())) == ref
    assert W.is_strongly_connected(n2, src, dst)


def test_frontend_errors(T):
    with pytest.raises(T.TacosError):
        T.tacos_build_hierarchical([{"kind": "switch", "n": 4, "degree": 4, "bw": 120}])
    with pytest.raises(T.TacosError):
        T.tacos_build_hierarchical([{"kind": "switch", "n": 4, "degree": 3, "bw": 100}])  # 100 % 3 != 0
    with pytest.raises(T.TacosError):
        T.tacos_build_hierarchical([{"kind": "ring", "n": 1, "bw": 1}])
