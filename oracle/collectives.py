"""Collective pre/postconditions and relay masks for the oracle (TEST INFRASTRUCTURE ONLY).

SURVEY §8 row f2 (general pre/post collectives with relays).  Plain Python
loops, written from the paper's definitions:

  * P:L70 Fig. CollectiveDefinition / P:L89 (§II.A): a collective is a
    precondition (which NPU holds which chunk at the start) and a
    postcondition (which NPU must hold which chunk at the end).
      - Broadcast from root: root holds chunks 0..k-1; every NPU requires them.
      - Scatter from root: root holds all N*k chunks; NPU x requires its own
        chunks x*k .. x*k+k-1 (the root keeps everything).
      - Gather to root: NPU x holds its own chunks; root requires all N*k.
  * P:L284 (§VII.A, Fig. CombiningCollective): a combining collective is the
    inverse of its non-combining counterpart: Reduce = reversed Broadcast; the
    paper pairs Gather with Scatter the same way (Table V).
  * Relays (reading R22): the paper's Scatter on the TEN
    (Fig. CollectiveOnTEN: "chunk 4 was transmitted from NPU 1 to
    2 at timestep 0" although NPU 2 does not require chunk 4) forwards chunks
    through NPUs that do not require them.  The greedy rule allows link s -> d
    to carry chunk c when d requires c, or when d is one hop closer than s to
    some NPU that requires c and does not hold it at the start (hop distance
    in G; R22).
  * Multi-tenant (Table VI): several collectives on one network at
    once = the union of their pre/postconditions over disjoint chunk ranges.
    A Reduce tenant inside such a merged forward search is scheduled as the
    Gather of its N partial chunks (reading R23).
"""
from __future__ import annotations

from collections import deque
from typing import List, Sequence, Tuple

import numpy as np


def _bits(n: int, C: int) -> np.ndarray:
    return np.zeros((n, (C + 31) // 32), dtype=np.uint32)


def _set(a: np.ndarray, x: int, c: int) -> None:
    a[x, c >> 5] |= np.uint32(1 << (c & 31))


def _get(a: np.ndarray, x: int, c: int) -> bool:
    return bool((int(a[x, c >> 5]) >> (c & 31)) & 1)


def named_bits(kind: str, n: int, k: int, root: int) -> Tuple[int, np.ndarray, np.ndarray]:
    """(C, pre, post) of BROADCAST / SCATTER / GATHER."""
    if not 0 <= root < n:
        raise ValueError("root out of range")
    if kind == "BROADCAST":
        C = k
        pre, post = _bits(n, C), _bits(n, C)
        for c in range(C):
            _set(pre, root, c)
            for x in range(n):
                _set(post, x, c)
        return C, pre, post
    C = n * k
    pre, post = _bits(n, C), _bits(n, C)
    if kind == "SCATTER":
        for c in range(C):
            _set(pre, root, c)
            _set(post, root, c)
            _set(post, c // k, c)
        return C, pre, post
    if kind == "GATHER":
        for c in range(C):
            _set(pre, c // k, c)
            _set(post, c // k, c)
            _set(post, root, c)
        return C, pre, post
    raise ValueError(kind)


def dual(kind: str) -> str:
    """the non-combining collective whose inverse (on G^T) gives `kind`."""
    return {"REDUCE": "BROADCAST", "GATHER": "SCATTER"}[kind]


def hop_distance_to(n: int, src: Sequence[int], dst: Sequence[int], targets: Sequence[int]) -> List[int]:
    """Hops from every NPU to the nearest target along the directed links (BFS
    from the targets over reversed links); -1 when no target is reachable."""
    into: List[List[int]] = [[] for _ in range(n)]
    for s, d in zip(src, dst):
        into[int(d)].append(int(s))
    dist = [-1] * n
    q = deque()
    for x in targets:
        if dist[x] < 0:
            dist[x] = 0
            q.append(x)
    while q:
        y = q.popleft()
        for x in into[y]:
            if dist[x] < 0:
                dist[x] = dist[y] + 1
                q.append(x)
    return dist


def relay_allow(n: int, src: Sequence[int], dst: Sequence[int], C: int, pre: np.ndarray,
                post: np.ndarray) -> np.ndarray:
    """allow[l] = post[dst_l] plus the chunks c that dst_l may relay: dst_l does
    not require c and lies on a shortest path from src_l to some NPU that
    requires c and lacks it at the start, i.e. is one hop closer than src_l to
    that NPU (R22).  L x ceil(C/32) u32 words."""
    pre = np.asarray(pre, dtype=np.uint32).reshape(n, -1)
    post = np.asarray(post, dtype=np.uint32).reshape(n, -1)
    L = len(src)
    allow = np.zeros((L, (C + 31) // 32), dtype=np.uint32)
    for l in range(L):
        allow[l] = post[int(dst[l])]
    for c in range(C):
        req = [x for x in range(n) if _get(post, x, c) and not _get(pre, x, c)]
        if not req:
            continue
        if all(_get(post, x, c) for x in range(n)):
            continue  # no NPU can relay c
        for r in req:
            dist = hop_distance_to(n, src, dst, [r])
            for l in range(L):
                s, d = int(src[l]), int(dst[l])
                if not _get(post, d, c) and dist[d] >= 0 and dist[s] == dist[d] + 1:
                    allow[l, c >> 5] |= np.uint32(1 << (c & 31))
    return allow


def multi_tenant(n: int, tenants: Sequence[Tuple[str, int, int]]) -> Tuple[int, np.ndarray, np.ndarray, List[int]]:
    """Union of tenants (kind, root, k) over disjoint chunk ranges.
    kinds: AG, BROADCAST, SCATTER, GATHER, REDUCE (as the Gather of its partial
    chunks, R23).  Returns (C, pre, post, first chunk of each tenant)."""
    parts = []
    for kind, root, k in tenants:
        if kind == "AG":
            C = n * k
            pre, post = _bits(n, C), _bits(n, C)
            for c in range(C):
                _set(pre, c // k, c)
                for x in range(n):
                    _set(post, x, c)
        else:
            C, pre, post = named_bits("GATHER" if kind == "REDUCE" else kind, n, k, root)
        parts.append((C, pre, post))
    C_tot = sum(p[0] for p in parts)
    pre_all, post_all = _bits(n, C_tot), _bits(n, C_tot)
    base, firsts = 0, []
    for C, pre, post in parts:
        firsts.append(base)
        for x in range(n):
            for c in range(C):
                if _get(pre, x, c):
                    _set(pre_all, x, base + c)
                if _get(post, x, c):
                    _set(post_all, x, base + c)
        base += C
    return C_tot, pre_all, post_all, firsts
