"""Topology and workload generators (inputs only; see package docstring).

Canonical link-id order: NPU ids of a torus / mesh are
``x + X*(y + Y*z)``; links are emitted node by node in id order, and per node in
the direction order +x, -x, +y, -y, +z, -z, skipping absent neighbours (mesh
borders) and duplicate neighbours (a torus dimension of size 2).  The same
arrays feed the oracle and the CUDA library, so both see identical link ids.

Units: alpha in integer ns, bandwidth in integer bytes/ns (= decimal GB/s,
SURVEY R6), chunk size in bytes (MiB/KiB).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Sequence, Tuple

import numpy as np

ALPHA_NS = 500  # P:L107 "alpha=0.5us"
MiB = 1 << 20
KiB = 1 << 10


@dataclass
class Topology:
    n_npus: int
    src: np.ndarray  # int32 [L]
    dst: np.ndarray  # int32 [L]
    alpha_ns: np.ndarray  # uint32 [L]
    bw: np.ndarray  # uint32 [L] bytes per ns
    name: str = ""

    @property
    def n_links(self) -> int:
        return int(self.src.shape[0])

    def links(self) -> List[Tuple[int, int, int, int]]:
        return list(zip(self.src.tolist(), self.dst.tolist(), self.alpha_ns.tolist(), self.bw.tolist()))


@dataclass
class Workload:
    name: str
    topo: Topology
    chunks_per_npu: int
    chunk_bytes: int
    collective: str  # "AG" or "AR"
    n_seeds: int
    base_seed: int = 0
    time_unit_ns: int = 1
    note: str = ""
    extra: dict = field(default_factory=dict)


def _mk(n: int, links: Sequence[Tuple[int, int, int, int]], name: str) -> Topology:
    if len(links) == 0:
        a = np.zeros(0, np.int64)
        return Topology(n, a.astype(np.int32), a.astype(np.int32), a.astype(np.uint32), a.astype(np.uint32), name)
    arr = np.asarray(links, dtype=np.int64)
    return Topology(
        n_npus=n,
        src=arr[:, 0].astype(np.int32),
        dst=arr[:, 1].astype(np.int32),
        alpha_ns=arr[:, 2].astype(np.uint32),
        bw=arr[:, 3].astype(np.uint32),
        name=name,
    )


def uni_ring(p: int, bw: int = 100, alpha: int = ALPHA_NS) -> Topology:
    """Uni-directional ring i -> i+1 (Fig. TenDefinition)."""
    return _mk(p, [(i, (i + 1) % p, alpha, bw) for i in range(p)], f"uni_ring{p}")


def bi_ring(p: int, bw: int = 100, alpha: int = ALPHA_NS) -> Topology:
    """Bi-directional ring; per node +1 then -1 (duplicates skipped for p=2)."""
    links = []
    for i in range(p):
        seen = set()
        for j in ((i + 1) % p, (i - 1) % p):
            if j != i and j not in seen:
                seen.add(j)
                links.append((i, j, alpha, bw))
    return _mk(p, links, f"bi_ring{p}")


def path(p: int, bw: int = 100, alpha: int = ALPHA_NS) -> Topology:
    """1-D mesh (bidirectional path)."""
    links = []
    for i in range(p):
        if i + 1 < p:
            links.append((i, i + 1, alpha, bw))
        if i - 1 >= 0:
            links.append((i, i - 1, alpha, bw))
    return _mk(p, links, f"path{p}")


def fully_connected(n: int, bw: int = 100, alpha: int = ALPHA_NS) -> Topology:
    return _mk(n, [(i, j, alpha, bw) for i in range(n) for j in range(n) if j != i], f"fc{n}")


def _grid(dims: Sequence[int], wrap: bool, bws: Sequence[int], alpha: int, name: str) -> Topology:
    dims = list(dims)
    nd = len(dims)
    n = int(np.prod(dims))
    strides = [int(np.prod(dims[:i])) for i in range(nd)]
    links = []
    for node in range(n):
        coord = [(node // strides[i]) % dims[i] for i in range(nd)]
        seen = set()
        for dim in range(nd):
            for step in (+1, -1):
                c = coord[dim] + step
                if wrap:
                    c %= dims[dim]
                elif c < 0 or c >= dims[dim]:
                    continue
                nb = node + (c - coord[dim]) * strides[dim]
                if nb == node or nb in seen:
                    continue
                seen.add(nb)
                links.append((node, nb, alpha, bws[dim]))
    return _mk(n, links, name)


def mesh2d(x: int, y: int, bw_x: int = 100, bw_y: int = 100, alpha: int = ALPHA_NS) -> Topology:
    return _grid([x, y], False, [bw_x, bw_y], alpha, f"mesh{x}x{y}")


def torus(dims: Sequence[int], bw: int = 100, alpha: int = ALPHA_NS) -> Topology:
    return _grid(list(dims), True, [bw] * len(dims), alpha, "torus" + "x".join(map(str, dims)))


def hypercube(d: int, bw: int = 100, alpha: int = ALPHA_NS) -> Topology:
    n = 1 << d
    return _mk(n, [(i, i ^ (1 << b), alpha, bw) for i in range(n) for b in range(d)], f"hypercube{d}")


def switch_hypercube_hybrid(groups: int = 16, group_size: int = 16, bw_intra: int = 20, bw_inter: int = 25,
                            alpha: int = ALPHA_NS) -> Topology:
    """Config 5 base graph: per group a switch unwound degree-max (= FC, P:L185-187,
    P:L289), groups joined as a hypercube on the group id.
    Per node: intra-group links to members j != i in increasing j, then one
    inter-group link per hypercube dimension b (group g -> g ^ (1<<b), same member)."""
    assert groups & (groups - 1) == 0
    d = groups.bit_length() - 1
    links = []
    for g in range(groups):
        for i in range(group_size):
            node = g * group_size + i
            for j in range(group_size):
                if j != i:
                    links.append((node, g * group_size + j, alpha, bw_intra))
            for b in range(d):
                links.append((node, (g ^ (1 << b)) * group_size + i, alpha, bw_inter))
    return _mk(groups * group_size, links, f"switch{group_size}x{groups}_hypercube")


def ring_fc_switch(ring: int = 2, fc: int = 4, switch: int = 64, bw_ring: int = 200, bw_fc: int = 100,
                   bw_switch: int = 50, alpha: int = ALPHA_NS) -> Topology:
    """The paper's scalability system Ring_FullyConnected_Switch ("3D
    topology of Ring_FullyConnected_Switch, node size 2x4, 200_100_50 GB/s",
    P:L289 "degree-max unwinding for scale-up switches and degree-1 for
    scale-out"): NPU id = r + ring*(f + fc*s); per NPU: ring link(s), FC links,
    then the scale-out switch unwound with degree 1 (a uni-directional ring)."""
    n = ring * fc * switch
    links = []
    for x in range(n):
        r, f, s = x % ring, (x // ring) % fc, x // (ring * fc)
        base_r, base_f = x - r, x - f * ring
        links.append((x, base_r + (r + 1) % ring, alpha, bw_ring))
        if ring > 2:
            links.append((x, base_r + (r - 1) % ring, alpha, bw_ring))
        for g in range(fc):
            if g != f:
                links.append((x, base_f + g * ring, alpha, bw_fc))
        links.append((x, x + (((s + 1) % switch) - s) * ring * fc, alpha, bw_switch))
    return _mk(n, links, f"ring{ring}_fc{fc}_switch{switch}")


def is_strongly_connected(n: int, src: np.ndarray, dst: np.ndarray) -> bool:
    """Plain BFS from node 0 on G and on G^T."""
    if n <= 1:
        return True
    for a, b in ((src, dst), (dst, src)):
        adj = [[] for _ in range(n)]
        for s, t in zip(a.tolist(), b.tolist()):
            adj[s].append(t)
        seen = [False] * n
        seen[0] = True
        stack = [0]
        while stack:
            u = stack.pop()
            for v in adj[u]:
                if not seen[v]:
                    seen[v] = True
                    stack.append(v)
        if not all(seen):
            return False
    return True


def remove_undirected_links(topo: Topology, fraction: float, seed: int, max_tries: int = 1000) -> Tuple[Topology, np.ndarray]:
    """Fail ``round(fraction * #undirected)`` physical links (both directions),
    chosen by a seeded draw, re-drawn until the graph stays strongly connected
    (P:L428 re-synthesis on the reduced topology)."""
    pairs = {}
    for idx, (s, d) in enumerate(zip(topo.src.tolist(), topo.dst.tolist())):
        key = (min(s, d), max(s, d))
        pairs.setdefault(key, []).append(idx)
    und = sorted(k for k, v in pairs.items() if len(v) == 2)
    n_fail = int(round(fraction * len(und)))
    rng = np.random.default_rng(seed)
    for _ in range(max_tries):
        pick = rng.choice(len(und), size=n_fail, replace=False)
        drop = set()
        for i in pick.tolist():
            drop.update(pairs[und[i]])
        keep = np.array([i for i in range(topo.n_links) if i not in drop], dtype=np.int64)
        if is_strongly_connected(topo.n_npus, topo.src[keep], topo.dst[keep]):
            failed = np.array(sorted(und[i] for i in pick.tolist()), dtype=np.int64)
            return (
                Topology(topo.n_npus, topo.src[keep].copy(), topo.dst[keep].copy(), topo.alpha_ns[keep].copy(),
                         topo.bw[keep].copy(), topo.name + f"_fail{n_fail}"),
                failed,
            )
    raise RuntimeError("could not draw a strongly connected failure set")


def random_strongly_connected(n: int, n_links: int, seed: int, bws: Sequence[int] = (100,), alphas: Sequence[int] = (0,)) -> Topology:
    """Random strongly connected digraph: a random Hamiltonian cycle plus random
    extra arcs, shuffled link order.  Used for brute-force pins."""
    rng = np.random.default_rng(seed)
    assert n >= 2 and n <= n_links <= n * (n - 1)
    perm = rng.permutation(n).tolist()
    arcs = {(perm[i], perm[(i + 1) % n]) for i in range(n)}
    if n == 2:
        arcs = {(0, 1), (1, 0)}
    cands = [(a, b) for a in range(n) for b in range(n) if a != b and (a, b) not in arcs]
    rng.shuffle(cands)
    for a in cands[: max(0, n_links - len(arcs))]:
        arcs.add(tuple(a))
    arcs = sorted(arcs)
    order = rng.permutation(len(arcs)).tolist()
    links = []
    for i in order:
        a, b = arcs[i]
        links.append((a, b, int(rng.choice(alphas)), int(rng.choice(bws))))
    return _mk(n, links, f"rand{n}_{len(arcs)}_{seed}")


def transpose(topo: Topology) -> Topology:
    """G^T keeping link ids (link j := dst_j -> src_j)."""
    return Topology(topo.n_npus, topo.dst.copy(), topo.src.copy(), topo.alpha_ns.copy(), topo.bw.copy(), topo.name + "_T")


# ----------------------------------------------------------------------------
# The five BASELINE.json configs
# ----------------------------------------------------------------------------

def config(i: int) -> Workload:
    if i == 1:
        return Workload("c1_uni_ring4_ag", uni_ring(4, 100), 1, 1 * MiB, "AG", 1,
                        note="4-NPU uni ring All-Gather, 1 chunk/NPU, uniform alpha/beta (hand-checkable)")
    if i == 2:
        return Workload("c2_torus8x8_ar", torus([8, 8], 100), 4, 1 * MiB, "AR", 64,
                        note="2D torus 8x8, AR, 4 chunks/NPU, 1 MiB chunks")
    if i == 3:
        return Workload("c3_torus8x8x8_ar", torus([8, 8, 8], 100), 1, 1 * MiB, "AR", 64,
                        note="3D torus 8x8x8 (512 NPUs), AR, 64 seeds batched")
    if i == 4:
        return Workload("c4_mesh32x32_hetero_ar", mesh2d(32, 32, 200, 100), 8, 128 * KiB, "AR", 16,
                        note="2D mesh 32x32, X 200 / Y 100 B/ns, AR, 8 chunks/NPU of 128 KiB")
    if i == 5:
        base = switch_hypercube_hybrid(16, 16, 20, 25)
        topo, failed = remove_undirected_links(base, 0.05, seed=5)
        return Workload("c5_switch_hypercube_fail5_ar", topo, 1, 1 * MiB, "AR", 256,
                        note="16 x FC(16) switch groups + 4-D hypercube, 5% undirected links failed, AR, 256 seeds",
                        extra={"failed_undirected": failed.tolist()})
    if i == 6 or i == "ctx":
        return Workload("ctx_ring2_fc4_switch64_ar", ring_fc_switch(2, 4, 64, 200, 100, 50), 1, 1 * MiB, "AR", 64,
                        note="paper's 512-NPU Ring(2) x FC(4) x Switch(64, d=1), 200/100/50 GB/s (P:L288-289, "
                             "P:L354); asymmetric: the RS is searched on G^T")
    raise ValueError(i)


CONFIGS = (1, 2, 3, 4, 5)
