"""Independent schedule checker for tests.

Shares nothing with the oracle or the product: a plain replay of a list of
sends against the TEN semantics: a send occupies its link on
[t_start, t_end) (R8), departs only with an arrived chunk, and the
postcondition must hold at the end.  The greedy-specific checks
(maximality, shorter-link-first) reconstruct the event
times from the schedule itself.
"""
from __future__ import annotations

from collections import defaultdict
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np


def check(n: int, src: Sequence[int], dst: Sequence[int], w: Sequence[int], sends: np.ndarray,
          pre: Sequence[set], post: Sequence[set], greedy: bool = True) -> Dict[str, object]:
    """Return a dict of violation lists (all empty = clean) plus T."""
    src = [int(x) for x in src]
    dst = [int(x) for x in dst]
    w = [int(x) for x in w]
    v: Dict[str, list] = defaultdict(list)
    recs = [tuple(int(r[f]) for f in ("chunk", "src", "dst", "link", "t_start", "t_end")) for r in sends]
    # link existence + duration
    for i, (c, a, b, l, t0, t1) in enumerate(recs):
        if not (0 <= l < len(src)) or src[l] != a or dst[l] != b:
            v["no_such_link"].append(i)
            continue
        if t1 - t0 != w[l]:
            v["wrong_duration"].append(i)
    # link intervals disjoint
    by_link = defaultdict(list)
    for i, (c, a, b, l, t0, t1) in enumerate(recs):
        by_link[l].append((t0, t1, i))
    for l, iv in by_link.items():
        iv.sort()
        for (a0, a1, _), (b0, b1, j) in zip(iv, iv[1:]):
            if b0 < a1:
                v["link_overlap"].append(j)
    # arrival times: arrive[(c, x)] = time x holds c
    arrive: Dict[Tuple[int, int], int] = {}
    for x in range(n):
        for c in pre[x]:
            arrive[(c, x)] = 0
    for i, (c, a, b, l, t0, t1) in sorted(enumerate(recs), key=lambda e: e[1][5]):
        if (c, b) in arrive:  # already held (pre) or delivered before
            v["duplicate_delivery"].append(i)
        else:
            arrive[(c, b)] = t1
    for i, (c, a, b, l, t0, t1) in enumerate(recs):
        ta = arrive.get((c, a))
        if ta is None or ta > t0:
            v["unheld_at_depart"].append(i)
    for x in range(n):
        for c in post[x]:
            if (c, x) not in arrive:
                v["post_unmet"].append((c, x))
    T = max((r[5] for r in recs), default=0)
    if greedy:
        _check_greedy(n, src, dst, w, recs, pre, post, arrive, v)
    out: Dict[str, object] = {k: val for k, val in v.items()}
    out["T"] = T
    return out


def _check_greedy(n, src, dst, w, recs, pre, post, arrive, v):
    """Maximality + shorter-link-first at every event."""
    events = sorted({0} | {r[5] for r in recs})
    T = max((r[5] for r in recs), default=0)
    starts = defaultdict(dict)  # t -> link -> chunk
    for (c, a, b, l, t0, t1) in recs:
        starts[t0][l] = c
    for t in events:
        if t >= T:
            continue
        held = [set(c for c in range(_nchunks(post)) if arrive.get((c, x), None) is not None and arrive[(c, x)] <= t)
                for x in range(n)]
        # in flight towards x at t (sent before t, arriving after t)
        pend = [set() for _ in range(n)]
        busy = set()
        for (c, a, b, l, t0, t1) in recs:
            if t0 < t < t1:
                pend[b].add(c)
                busy.add(l)
        claimed_now = defaultdict(dict)  # x -> chunk -> link
        for l, c in starts[t].items():
            claimed_now[dst[l]][c] = l
        for l in range(len(src)):
            if l in busy or l in starts[t]:
                continue
            a, b = src[l], dst[l]
            cand = (held[a] & set(post[b])) - held[b] - pend[b]
            for c in cand:
                if c not in claimed_now[b]:
                    v["not_maximal"].append((t, l, c))
                elif w[claimed_now[b][c]] > w[l]:
                    v["not_shorter_first"].append((t, l, c))


def _nchunks(post):
    return max((max(p) + 1 for p in post if p), default=0)


def clean(rep) -> bool:
    return all(len(val) == 0 for k, val in rep.items() if k != "T")


def ag_sets(n: int, k: int):
    pre = [set(range(x * k, x * k + k)) for x in range(n)]
    post = [set(range(n * k)) for _ in range(n)]
    return pre, post
