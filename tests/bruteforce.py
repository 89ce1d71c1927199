"""Exhaustive optimum for tiny All-Gather instances.

Independent of the oracle: it searches EVERY congestion-free schedule in the
discrete TEN with time unit 1 (TEN edges (u_t, v_{t+w})), where at
every time step each free link either idles or sends one chunk its source holds
(arrived) and its destination needs, lacks and is not already
receiving (no duplicate in-flight copies; R4).  Idling stays in the search:
waiting for a better chunk can beat sending now (E7).  Returns T_opt, the
minimum finishing time; TACOS-Greedy (a heuristic) must never beat it.
"""
from __future__ import annotations

import itertools
from functools import lru_cache
from typing import List, Optional, Sequence, Tuple


def optimum(n: int, links: Sequence[Tuple[int, int, int]], pre: Sequence[int], post: Sequence[int],
            t_max: int = 32, relays: bool = False) -> Optional[int]:
    """links: (src, dst, w) with integer w >= 1.  pre/post: per-NPU chunk bitmasks.
    relays=True: a link may also carry a chunk its destination does not require
    (any relay at all, a superset of the greedy's shortest-path relays, R22).
    Returns the minimum T or None if not reachable within t_max."""
    L = len(links)
    INF = 10 ** 9
    # all-pairs shortest w-distance for the admissible lower bound
    dist = [[INF] * n for _ in range(n)]
    for i in range(n):
        dist[i][i] = 0
    for s, d, w in links:
        dist[s][d] = min(dist[s][d], w)
    for k in range(n):
        for i in range(n):
            for j in range(n):
                if dist[i][k] + dist[k][j] < dist[i][j]:
                    dist[i][j] = dist[i][k] + dist[k][j]
    n_chunks = max((p.bit_length() for p in list(pre) + list(post)), default=0)
    post_t = tuple(post)
    all_chunks = (1 << n_chunks) - 1

    def lower_bound(held, inflight):
        lb = 0
        # earliest time chunk c can be at some NPU: 0 where held, rem where in flight
        avail = {}
        for l, f in enumerate(inflight):
            if f is not None:
                c, rem = f
                key = (c, links[l][1])
                avail[key] = min(avail.get(key, INF), rem)
        for x in range(n):
            need = post_t[x] & ~held[x]
            c = 0
            while need:
                if need & 1:
                    best = INF
                    for y in range(n):
                        if (held[y] >> c) & 1:
                            best = min(best, dist[y][x])
                        elif (c, y) in avail:
                            best = min(best, avail[(c, y)] + dist[y][x])
                    if best >= INF:
                        return INF
                    lb = max(lb, best)
                need >>= 1
                c += 1
        return lb

    @lru_cache(maxsize=None)
    def feasible(held, inflight, budget):
        # state is at an instant, after arrivals; budget = time units left
        if all((post_t[x] & ~held[x]) == 0 for x in range(n)):
            return True
        if budget <= 0:
            return False
        if lower_bound(held, inflight) > budget:
            return False
        incoming = [0] * n  # chunks already in flight towards x
        for l, f in enumerate(inflight):
            if f is not None:
                incoming[links[l][1]] |= 1 << f[0]
        options: List[List[Optional[int]]] = []
        for l, (s, d, w) in enumerate(links):
            if inflight[l] is not None:
                options.append([None])
                continue
            useful = held[s] & (all_chunks if relays else post_t[d]) & ~held[d] & ~incoming[d]
            opts: List[Optional[int]] = [None]
            c = 0
            while useful:
                if useful & 1:
                    opts.append(c)
                useful >>= 1
                c += 1
            options.append(opts)
        any_inflight = any(f is not None for f in inflight)
        for choice in itertools.product(*options):
            if not any_inflight and all(c is None for c in choice):
                continue  # pure waiting with nothing in flight changes nothing
            # at most one copy of a chunk towards each destination
            seen = set()
            ok = True
            for l, c in enumerate(choice):
                if c is not None:
                    key = (c, links[l][1])
                    if key in seen:
                        ok = False
                        break
                    seen.add(key)
            if not ok:
                continue
            new_inf = list(inflight)
            for l, c in enumerate(choice):
                if c is not None:
                    new_inf[l] = (c, links[l][2])
            # advance one time unit; arrivals land at the next instant
            nh = list(held)
            nxt = []
            for l, f in enumerate(new_inf):
                if f is None:
                    nxt.append(None)
                    continue
                c, rem = f
                rem -= 1
                if rem == 0:
                    nh[links[l][1]] |= 1 << c
                    nxt.append(None)
                else:
                    nxt.append((c, rem))
            if feasible(tuple(nh), tuple(nxt), budget - 1):
                return True
        return False

    held0 = tuple(pre)
    inf0 = tuple([None] * L)
    for T in range(0, t_max + 1):
        if feasible(held0, inf0, T):
            return T
    return None


def allgather_masks(n: int, k: int) -> Tuple[List[int], List[int]]:
    C = n * k
    pre = [sum(1 << (x * k + j) for j in range(k)) for x in range(n)]
    post = [(1 << C) - 1] * n
    return pre, post
