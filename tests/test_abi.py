"""CPU tests of the C ABI boundary (no compute on a GPU): the library loads and
exports every symbol include/tacos.h declares; host-side validation, cost
quantization, symmetry / connectivity, and the tacos_eval verifier."""
import os
import re

import numpy as np
import pytest

import oracle
import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def T():
    from paper_2304_05301_b200 import build

    build.build()
    import paper_2304_05301_b200 as T

    T.load_library()
    return T


def declared_functions():
    src = open(os.path.join(ROOT, "include", "tacos.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tacos_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(T):
    names = declared_functions()
    assert len(names) >= 30
    lib = T.load_library()
    for n in names:
        assert hasattr(lib, n), n
        assert n in T.SIGNATURES, f"binding lacks {n}"
    assert lib.tacos_abi_version() == 1


def test_no_cpu_fallback_without_device(T):
    """The synthesis entry points must fail loudly (TACOS_E_CUDA) when no GPU
    is visible -- never compute on the host."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    t = T.Topology.from_workload_topology(W.uni_ring(4))
    with pytest.raises(T.TacosError) as e:
        T.synthesize(t, "AG", 1, 1 << 20, 1)
    assert e.value.code == T.TACOS_E_CUDA


@pytest.mark.parametrize("case,code", [
    ("self_loop", -2), ("dup", -2), ("range", -2), ("bw0", -2), ("n1", -1),
])
def test_topology_validation(T, case, code):
    args = {
        "self_loop": (3, [0, 1, 2], [1, 1, 0], [1, 1, 1], [1, 1, 1]),
        "dup": (3, [0, 0, 1], [1, 1, 2], [1, 1, 1], [1, 1, 1]),
        "range": (3, [0, 5], [1, 2], [1, 1], [1, 1]),
        "bw0": (2, [0, 1], [1, 0], [1, 1], [1, 0]),
        "n1": (1, [0], [0], [1], [1]),
    }[case]
    with pytest.raises(T.TacosError) as e:
        T.Topology(*args)
    assert e.value.code == code


def test_link_costs_match_oracle(T):
    for topo, nb, f in [(W.config(4).topo, 128 << 10, 1), (W.config(5).topo, 1 << 20, 1),
                        (W.random_strongly_connected(6, 15, 1, bws=(3, 7, 100), alphas=(0, 13, 999)), 12345, 7)]:
        t = T.Topology.from_workload_topology(topo)
        assert np.array_equal(t.link_costs(nb, f).astype(np.uint64), oracle.link_costs(topo, nb, f))


def test_cost_errors(T):
    t = T.Topology(2, [0, 1], [1, 0], [0, 0], [5, 5])
    with pytest.raises(T.TacosError) as e:
        t.link_costs(0)
    assert e.value.code == T.TACOS_E_TOPOLOGY
    t2 = T.Topology(2, [0, 1], [1, 0], [4_000_000_000, 1], [1, 1])
    with pytest.raises(T.TacosError) as e:
        t2.link_costs(2**62)
    assert e.value.code == T.TACOS_E_OVERFLOW


def test_symmetry_and_connectivity(T):
    assert T.Topology.from_workload_topology(W.torus([4, 4])).is_symmetric(1 << 20)
    assert not T.Topology.from_workload_topology(W.uni_ring(5)).is_symmetric(1 << 20)
    # config 4: X and Y costs differ but each cable is symmetric
    assert T.Topology.from_workload_topology(W.config(4).topo).is_symmetric(128 << 10)
    assert T.Topology.from_workload_topology(W.config(5).topo).strongly_connected
    # a path directed one way is not strongly connected
    assert not T.Topology(3, [0, 1], [1, 2], [1, 1], [1, 1]).strongly_connected


# --------------------------------------------------------------------------
# tacos_eval against oracle schedules and mutations of them
# --------------------------------------------------------------------------
@pytest.mark.parametrize("coll", ["AG", "RS", "AR"])
@pytest.mark.parametrize("name", ["torus44", "uni5", "hetero"])
def test_eval_accepts_oracle_schedules(T, coll, name):
    topo = {"torus44": W.torus([4, 4]), "uni5": W.uni_ring(5), "hetero": W.mesh2d(3, 4, 200, 100)}[name]
    syn = oracle.synthesize(topo, 2, 1 << 20, coll, [0, 1])
    t = T.Topology.from_workload_topology(topo)
    rep = T.evaluate(t, syn.sends, coll, 2, 1 << 20)
    assert rep["n_violations"] == 0, rep
    assert rep["T"] == syn.T
    if coll == "AR":
        assert rep["T_rs"] == syn.T_rs


def test_eval_flags_mutations(T):
    topo = W.torus([4, 4])
    syn = oracle.synthesize(topo, 1, 1 << 20, "AG", [3])
    t = T.Topology.from_workload_topology(topo)
    base = syn.sends.copy()

    def rep_of(s):
        return T.evaluate(t, s, "AG", 1, 1 << 20)

    s = base[1:]  # drop one send -> post unmet
    assert rep_of(s)["post_unmet"] == 1
    s = base.copy()
    s[5]["t_end"] += 1  # wrong duration
    assert rep_of(s)["wrong_duration"] >= 1
    s = base.copy()
    s[7]["link"] = (s[7]["link"] + 1) % topo.n_links  # endpoints no longer match the link
    assert rep_of(s)["no_such_link"] == 1
    s = np.concatenate([base, base[:1]])  # duplicate delivery + overlap on that link
    r = rep_of(s)
    assert r["duplicate_delivery"] == 1 and r["link_overlap"] == 1
    # departs before holding: move a relayed send earlier than its chunk's arrival
    relayed = [i for i, x in enumerate(base) if int(x["chunk"]) != int(x["src"])]
    s = base.copy()
    i = relayed[-1]
    s[i]["t_start"] = 0
    s[i]["t_end"] = int(s[i]["t_end"]) - int(base[i]["t_start"])
    assert rep_of(s)["unheld_at_depart"] >= 1


def test_multi_device_entry_points_without_gpu(T):
    """The multi-GPU entry points fail loudly without a device (no CPU fallback), and NCCL is
    resolved at run time (dlopen): the library reports the version it would use."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    t = T.Topology.from_workload_topology(W.torus([4, 4]))
    with pytest.raises(T.TacosError) as e:
        T.synthesize(t, "AR", 1, 1 << 20, 4, n_devices=2)
    assert e.value.code == T.TACOS_E_CUDA
    with pytest.raises(T.TacosError) as e:
        T.synthesize_batch([t, t], collective="AR", n_seeds=2, n_devices=2)
    assert e.value.code == T.TACOS_E_CUDA
    try:
        v = T.nccl_version()
    except T.TacosError as err:  # no NCCL on this host: the documented error
        assert err.code == T.TACOS_E_NCCL
    else:
        assert v >= 20000


def test_link_costs_wide_arithmetic(T):
    """a1: w = ceil((alpha * bw + n) / (bw * f)) exactly, on both sides of the
    64-bit numerator boundary (the library divides in 64 bits when alpha * bw + n fits, in 128
    bits otherwise), with the error codes for w = 0 and w >= 2^32 - 1; the expected values are
    the definition in Python integers."""
    rng = np.random.default_rng(5)
    M32, M64 = 2**32 - 1, 2**64 - 1
    cases = []
    for a in (0, 1, 7, M32, int(rng.integers(1, M32))):
        for b in (1, 3, M32, int(rng.integers(1, M32))):
            ab = a * b
            for n in (0, 1, M64 - ab, min(M64, M64 - ab + 1), 2**63, M64, int(rng.integers(0, 2**63))):
                if n > M64:
                    continue
                for f in (1, 2**31, M32):
                    cases.append((a, b, n, f))
    for a, b, n, f in cases:
        t = T.Topology(2, [0, 1], [1, 0], [a, a], [b, b])
        q = -(-(a * b + n) // (b * f))
        if q == 0:
            with pytest.raises(T.TacosError) as e:
                t.link_costs(n, f)
            assert e.value.code == T.TACOS_E_TOPOLOGY
        elif q >= M32:
            with pytest.raises(T.TacosError) as e:
                t.link_costs(n, f)
            assert e.value.code == T.TACOS_E_OVERFLOW
        else:
            assert t.link_costs(n, f).tolist() == [q, q], (a, b, n, f)
