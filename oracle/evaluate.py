"""Continuous-time evaluator and Ring / Direct baselines (TEST INFRASTRUCTURE
ONLY).  Plain Python with exact rational time (fractions),
written from the definitions, independent of the product's C++.

  * a send on link l lasts alpha_l + n / bw_l ns (unrounded);
  * links are exclusive and serve sends first come first served in the
    schedule's (t_start, array position) order ("queueing-based link
    congestion");
  * AG-type sends wait for their chunk at the source; RS-type sends (RS phase)
    wait for every RS send of that chunk into the source (a reduction is the
    mirror of a broadcast); an AR's AG phase starts after the RS phase
    (R10) and at the owner's reduced chunk;
  * baselines: logical ring over NPU ids, or direct all-to-all;
    every logical transfer routed on a shortest hop path found by BFS over
    out-links in link-id order (xy routing on a canonical mesh).
"""
from fractions import Fraction
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import SEND_DTYPE, link_costs


def evaluate(topo, sends: np.ndarray, collective: str, k: int, chunk_bytes: int) -> Tuple[Fraction, Fraction]:
    n, L = topo.n_npus, topo.n_links
    dur = [Fraction(int(a)) + Fraction(chunk_bytes, int(b)) for a, b in zip(topo.alpha_ns, topo.bw)]
    C = n * k
    recs = [tuple(int(r[f]) for f in ("chunk", "src", "dst", "link", "t_start")) for r in sends]
    order = sorted(range(len(recs)), key=lambda i: recs[i][4])  # stable: array position breaks ties
    n_rs = 0
    if collective == "AR":
        n_rs = len(recs) // 2
        by_tl = sorted(range(len(recs)), key=lambda i: (recs[i][4], recs[i][3]))
        rs_set = set(by_tl[:n_rs])
        order = [i for i in order if i in rs_set] + [i for i in order if i not in rs_set]
    elif collective == "RS":
        n_rs = len(recs)
    link_free = [Fraction(0)] * L
    rs_in = {}
    T_rs = Fraction(0)
    for i in order[:n_rs]:
        c, a, b, l, _ = recs[i]
        st = max(rs_in.get((a, c), Fraction(0)), link_free[l])
        en = st + dur[l]
        link_free[l] = en
        rs_in[(b, c)] = max(rs_in.get((b, c), Fraction(0)), en)
        T_rs = max(T_rs, en)
    avail = {}
    for c in range(C):
        o = c // k
        avail[(o, c)] = max(T_rs, rs_in.get((o, c), Fraction(0))) if collective == "AR" else Fraction(0)
    T = T_rs
    for i in order[n_rs:]:
        c, a, b, l, _ = recs[i]
        ready = avail[(a, c)]  # KeyError = departs before holding
        st = max(ready, link_free[l])
        en = st + dur[l]
        link_free[l] = en
        avail[(b, c)] = min(avail.get((b, c), en), en)
        T = max(T, en)
    return T, T_rs


def _bfs_paths(topo, s: int, transposed: bool):
    n = topo.n_npus
    out = [[] for _ in range(n)]
    for l in range(topo.n_links):
        a, b = int(topo.src[l]), int(topo.dst[l])
        if transposed:
            a, b = b, a
        out[a].append((l, b))  # link-id order
    parent = [None] * n
    seen = [False] * n
    seen[s] = True
    q = [s]
    for x in q:
        for l, y in out[x]:
            if not seen[y]:
                seen[y] = True
                parent[y] = (l, x)
                q.append(y)
    return parent


def _path(parent, s, d):
    hops = []
    x = d
    while x != s:
        l, px = parent[x]
        hops.append((l, px, x))
        x = px
    return hops[::-1]


def _ag(topo, k: int, alg: str, transposed: bool):
    n = topo.n_npus
    parents = [_bfs_paths(topo, s, transposed) for s in range(n)]
    out = []  # (chunk, a, b, link, key)
    if alg == "ring":
        # logical successor i+1 on G; on G^T (RS, mirrored back) i-1
        step = -1 if transposed else 1
        H = max(1, max(len(_path(parents[i], i, (i + step) % n)) for i in range(n)))
        for j in range(n - 1):
            for i in range(n):
                owner = (i - step * j) % n
                for h, (l, a, b) in enumerate(_path(parents[i], i, (i + step) % n)):
                    for q in range(k):
                        out.append((owner * k + q, a, b, l, j * H + h))
    else:
        for owner in range(n):
            for d in range(n):
                if d == owner:
                    continue
                for h, (l, a, b) in enumerate(_path(parents[owner], owner, d)):
                    for q in range(k):
                        out.append((owner * k + q, a, b, l, h))
    out.sort(key=lambda r: r[4])
    return out


def baseline(topo, alg: str, collective: str, k: int, chunk_bytes: int) -> np.ndarray:
    w = link_costs(topo, chunk_bytes)
    ag = _ag(topo, k, alg, False) if collective != "RS" else []
    rs = _ag(topo, k, alg, True) if collective != "AG" else []
    kmax = max((r[4] for r in rs), default=0)
    rows = []
    for (c, a, b, l, key) in reversed(rs):
        t0 = kmax - key
        rows.append((c, b, a, l, t0, t0 + int(w[l])))
    shift = kmax + 1 if rs else 0
    for (c, a, b, l, key) in ag:
        rows.append((c, a, b, l, key + shift, key + shift + int(w[l])))
    out = np.zeros(len(rows), dtype=SEND_DTYPE)
    for i, r in enumerate(rows):
        out[i] = r
    return out
