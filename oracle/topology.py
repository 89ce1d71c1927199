"""Topology front-end reference (TEST INFRASTRUCTURE ONLY).

Plain-loop definitions written from the paper, independent of the product's
C++ front-end (tacos_build_hierarchical / tacos_remove_npus):
  * switch unwinding with degree d (§IV.D): NPU n gets links
    n -> n+1, ..., n -> n+d (mod N); each keeps alpha, bandwidth / d; d = 1 also
    has a bi-directional ring variation at full bandwidth;
  * hierarchical composition Ring / FC / Switch / Path per dimension (P:L288
    "3D topology of Ring_FullyConnected_Switch");
  * NPU removal with dense renumbering (Table IV).
"""
from typing import Dict, List, Sequence, Tuple


def dim_links(kind: str, n: int, degree: int = 1, bidirectional: bool = False, alpha: int = 500,
              bw: int = 100) -> List[Tuple[int, int, int, int]]:
    links = []
    if kind == "ring":
        for i in range(n):
            links.append((i, (i + 1) % n, alpha, bw))
            if bidirectional and n > 2:
                links.append((i, (i - 1) % n, alpha, bw))
    elif kind == "fc":
        for i in range(n):
            for j in range(n):
                if i != j:
                    links.append((i, j, alpha, bw))
    elif kind == "switch":
        assert 1 <= degree <= n - 1 and bw % degree == 0
        if degree == 1 and bidirectional:
            return dim_links("ring", n, 1, True, alpha, bw)
        for i in range(n):
            for s in range(1, degree + 1):
                links.append((i, (i + s) % n, alpha, bw // degree))
    elif kind == "path":
        for i in range(n):
            if i + 1 < n:
                links.append((i, i + 1, alpha, bw))
            if i - 1 >= 0:
                links.append((i, i - 1, alpha, bw))
    else:
        raise ValueError(kind)
    return links


def hierarchical(dims: Sequence[Dict]) -> Tuple[int, List[Tuple[int, int, int, int]]]:
    """Product graph; NPU id = c0 + n0*(c1 + n1*(...)); per NPU, dimension by
    dimension, the dimension's links leaving the NPU's coordinate in order."""
    sizes = [d["n"] for d in dims]
    per = [dim_links(d["kind"], d["n"], d.get("degree", 1), bool(d.get("bidirectional", 0)), d.get("alpha_ns", 500),
                     d["bw"]) for d in dims]
    N = 1
    for s in sizes:
        N *= s
    out = []
    for x in range(N):
        coord, r = [], x
        for s in sizes:
            coord.append(r % s)
            r //= s
        stride = 1
        for i, s in enumerate(sizes):
            for (a, b, al, bw) in per[i]:
                if a == coord[i]:
                    out.append((x, x + (b - a) * stride, al, bw))
            stride *= s
    return N, out


def remove_npus(n: int, links: Sequence[Tuple[int, int, int, int]], removed: Sequence[int]):
    gone = set(removed)
    keep = [x for x in range(n) if x not in gone]
    nid = {x: i for i, x in enumerate(keep)}
    out = [(nid[a], nid[b], al, bw) for (a, b, al, bw) in links if a not in gone and b not in gone]
    return len(keep), out, keep
