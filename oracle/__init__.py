"""CPU oracle for TACOS-Greedy (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  It shares no code with
the CUDA product path (paper_2304_05301_b200/); neither imports the other.

Layers (PAPER.md = P:L<line>; SURVEY.md §8(c) readings = R<n>):
  * tacos_oracle.c (plain C, via ctypes): Philox4x32-10 (R2), link-cost
    quantization (a1), one greedy All-Gather synthesis per
    seed (a2-a6).
  * this file (numpy): inversion / All-Reduce composition and best-of-S
    (a7-a8; "Reduce-Scatter can be synthesized by simply inverting the
    topology-aware All-Gather ... All-Reduce is synthesized by running
    Reduce-Scatter followed by an All-Gather"; "choose the best
    algorithm among synthesized ones").
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tacos_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None
_lock = threading.Lock()

OK = 0
E_INVALID_ARG = -1
E_UNREACHABLE = -3
E_NOMEM = -5
E_OVERFLOW = -6
E_CAPACITY = -9

SEND_DTYPE = np.dtype(
    [("chunk", "<u4"), ("src", "<u4"), ("dst", "<u4"), ("link", "<u4"), ("t_start", "<u8"), ("t_end", "<u8")]
)
assert SEND_DTYPE.itemsize == 32


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C11)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-shared", "-fPIC", "-o", tmp, _SRC])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            l = ctypes.CDLL(build())
            u32p = ctypes.POINTER(ctypes.c_uint32)
            u64p = ctypes.POINTER(ctypes.c_uint64)
            i32p = ctypes.POINTER(ctypes.c_int32)
            l.oracle_link_cost.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint32, u64p]
            l.oracle_link_cost.restype = ctypes.c_int
            l.oracle_philox4x32_10.argtypes = [u32p, u32p, u32p]
            l.oracle_philox4x32_10.restype = None
            l.oracle_greedy.argtypes = [
                ctypes.c_int32, ctypes.c_int32, i32p, i32p, u64p, ctypes.c_uint32, ctypes.c_uint32, u32p, u32p,
                ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_uint64, u64p, u64p, u64p,
            ]
            l.oracle_greedy.restype = ctypes.c_int
            l.oracle_greedy_literal.argtypes = l.oracle_greedy.argtypes
            l.oracle_greedy_literal.restype = ctypes.c_int
            l.oracle_greedy_relay.argtypes = [
                ctypes.c_int32, ctypes.c_int32, i32p, i32p, u64p, ctypes.c_uint32, u32p, u32p, u32p,
                ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_uint64, u64p, u64p, u64p,
            ]
            l.oracle_greedy_relay.restype = ctypes.c_int
            _lib = l
    return _lib


def _p(a: np.ndarray, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str = ""):
        super().__init__(f"oracle error {code} {what}")
        self.code = code


# --------------------------------------------------------------------------
# R2 / P1
# --------------------------------------------------------------------------
def philox(ctr: Sequence[int], key: Sequence[int]) -> List[int]:
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    o = np.zeros(4, dtype=np.uint32)
    lib().oracle_philox4x32_10(_p(c, ctypes.c_uint32), _p(k, ctypes.c_uint32), _p(o, ctypes.c_uint32))
    return [int(x) for x in o]


# --------------------------------------------------------------------------
# a1
# --------------------------------------------------------------------------
def link_cost(alpha_ns: int, bw: int, chunk_bytes: int, f_ns: int = 1) -> int:
    w = ctypes.c_uint64(0)
    rc = lib().oracle_link_cost(alpha_ns, bw, chunk_bytes, f_ns, ctypes.byref(w))
    if rc != OK:
        raise OracleError(rc, "link_cost")
    return int(w.value)


def link_costs(topo, chunk_bytes: int, f_ns: int = 1) -> np.ndarray:
    return np.array([link_cost(int(a), int(b), chunk_bytes, f_ns) for a, b in zip(topo.alpha_ns, topo.bw)],
                    dtype=np.uint64)


# --------------------------------------------------------------------------
# a2-a6: one seed
# --------------------------------------------------------------------------
@dataclass
class GreedyResult:
    T: int
    sends: np.ndarray  # SEND_DTYPE, production order
    V: int
    D: int
    M: int
    E: int
    seed: int
    sigma: int
    X: int = 0  # cancelled sends (paper-literal variant: duplicates + replaced outdated transmissions)


def greedy(n_npus: int, src: np.ndarray, dst: np.ndarray, w: np.ndarray, n_chunks: int, k: int, seed: int,
           sigma: int = 0, pre: Optional[np.ndarray] = None, post: Optional[np.ndarray] = None,
           record: bool = True, literal: bool = False, allow: Optional[np.ndarray] = None) -> GreedyResult:
    """One TACOS-Greedy synthesis (SURVEY §8(c) pseudo-code); literal=True runs the
    paper-literal chunk-first variant with chunk replacement (row f1, reading R21);
    allow (L x ceil(C/32) words, CUSTOM only) = the chunks each link may carry,
    relays included (row f2, reading R22; see oracle/collectives.py)."""
    src = np.ascontiguousarray(src, dtype=np.int32)
    dst = np.ascontiguousarray(dst, dtype=np.int32)
    w = np.ascontiguousarray(w, dtype=np.uint64)
    Wd = (n_chunks + 31) // 32
    if pre is None:
        cap = n_chunks * (n_npus - 1)
        pre_p = post_p = None
    else:
        pre = np.ascontiguousarray(pre, dtype=np.uint32).reshape(n_npus, Wd)
        post = np.ascontiguousarray(post, dtype=np.uint32).reshape(n_npus, Wd)
        cap = int(sum(bin(int(x)).count("1") for x in (post & ~pre).ravel()))
        if allow is not None:  # relays: every (NPU, chunk) pair is delivered at most once
            cap = n_npus * n_chunks - int(sum(bin(int(x)).count("1") for x in pre.ravel()))
        pre_p, post_p = _p(pre, ctypes.c_uint32), _p(post, ctypes.c_uint32)
    sends = np.zeros(max(cap, 1), dtype=SEND_DTYPE)
    n_sends = ctypes.c_uint64(0)
    T = ctypes.c_uint64(0)
    stats = np.zeros(5, dtype=np.uint64)
    if allow is not None:
        if pre is None or literal:
            raise ValueError("allow masks need CUSTOM pre/post and the link-first variant")
        allow = np.ascontiguousarray(allow, dtype=np.uint32).reshape(src.shape[0], Wd)
        rc = lib().oracle_greedy_relay(
            n_npus, src.shape[0], _p(src, ctypes.c_int32), _p(dst, ctypes.c_int32), _p(w, ctypes.c_uint64),
            n_chunks, pre_p, post_p, _p(allow, ctypes.c_uint32), ctypes.c_uint64(seed & (2**64 - 1)), sigma,
            sends.ctypes.data if record else None, cap, ctypes.byref(n_sends), ctypes.byref(T),
            _p(stats, ctypes.c_uint64))
    else:
        fn = lib().oracle_greedy_literal if literal else lib().oracle_greedy
        rc = fn(
            n_npus, src.shape[0], _p(src, ctypes.c_int32), _p(dst, ctypes.c_int32), _p(w, ctypes.c_uint64),
            n_chunks, k, pre_p, post_p, ctypes.c_uint64(seed & (2**64 - 1)), sigma,
            sends.ctypes.data if record else None, cap, ctypes.byref(n_sends), ctypes.byref(T),
            _p(stats, ctypes.c_uint64),
        )
    if rc != OK:
        raise OracleError(rc, f"greedy seed={seed} sigma={sigma}")
    return GreedyResult(int(T.value), sends[: int(n_sends.value)] if record else sends[:0], int(stats[0]),
                        int(stats[1]), int(stats[2]), int(stats[3]), seed, sigma, int(stats[4]))


# --------------------------------------------------------------------------
# a7-a8: inversion, All-Reduce, best-of-S (R9-R11)
# --------------------------------------------------------------------------
def reverse_links(src: np.ndarray, dst: np.ndarray, w: np.ndarray) -> Optional[np.ndarray]:
    """rev[j] = id of link dst_j -> src_j if every link has a reverse with equal
    cost (G symmetric, R9); else None."""
    index = {(int(s), int(d)): j for j, (s, d) in enumerate(zip(src.tolist(), dst.tolist()))}
    rev = np.zeros(len(index), dtype=np.int64)
    for j, (s, d) in enumerate(zip(src.tolist(), dst.tolist())):
        r = index.get((d, s))
        if r is None or int(w[r]) != int(w[j]):
            return None
        rev[j] = r
    return rev


def mirror(sends: np.ndarray, T: int, src: np.ndarray, dst: np.ndarray, rev: Optional[np.ndarray]) -> np.ndarray:
    """Time-reverse a schedule: (c, a->b, t0, t1) -> (c, b->a, T-t1, T-t0)
    (P:L284 Fig. CombiningCollective: Reduce = reversed Broadcast).
    rev given: the input is on G and lands on the reverse link rev[j].
    rev None: the input is an AG on G^T (link j = dst_j -> src_j), and it lands
    on G's own link j (src_j -> dst_j)."""
    out = np.zeros(sends.shape[0], dtype=SEND_DTYPE)
    out["chunk"] = sends["chunk"]
    out["src"] = sends["dst"]
    out["dst"] = sends["src"]
    out["link"] = rev[sends["link"]] if rev is not None else sends["link"]
    out["t_start"] = np.uint64(T) - sends["t_end"]
    out["t_end"] = np.uint64(T) - sends["t_start"]
    return out


def canonical(sends: np.ndarray) -> np.ndarray:
    """Output order: ascending (t_start, link)."""
    order = np.lexsort((sends["link"], sends["t_start"]))
    return sends[order]


@dataclass
class Synthesis:
    collective: str
    T: int
    sends: np.ndarray
    seed: int  # winning AG seed
    rs_seed: int  # winning RS seed (== seed when G symmetric)
    T_ag: int
    T_rs: int
    seed_times: np.ndarray  # per seed collective time: AG T_AG(s), RS T_RS(s), AR T_RS(s) + T_AG(s)
    ag: List[GreedyResult]
    rs: List[GreedyResult]


NAMED = ("BROADCAST", "REDUCE", "SCATTER", "GATHER")


def synthesize(topo, chunks_per_npu: int, chunk_bytes: int, collective: str = "AR", seeds: Sequence[int] = (0,),
               time_unit_ns: int = 1, pre: Optional[np.ndarray] = None, post: Optional[np.ndarray] = None,
               threads: Optional[int] = None, record: bool = True, n_chunks: Optional[int] = None,
               literal: bool = False, relay: bool = False, root: int = 0) -> Synthesis:
    """Best-of-S TACOS-Greedy synthesis of AG / RS / AR (or CUSTOM with pre/post,
    collective 'CUSTOM', relays with relay=True), or of the named collectives of
    row f2: BROADCAST / SCATTER searched forward (Scatter with relays), REDUCE /
    GATHER as the inverse of BROADCAST / SCATTER on G^T, k chunks per
    NPU, `root`.  seeds are the 64-bit Philox keys; ties go to the lowest
    position in ``seeds`` (R11)."""
    from . import collectives as _coll

    n = topo.n_npus
    w = link_costs(topo, chunk_bytes, time_unit_ns)
    if collective in NAMED:
        fwd = collective if collective in ("BROADCAST", "SCATTER") else _coll.dual(collective)
        C, pre, post = _coll.named_bits(fwd, n, chunks_per_npu, root)
        relay = relay or fwd == "SCATTER"
    elif pre is None:
        C = n * chunks_per_npu
    else:
        if n_chunks is None:
            raise ValueError("CUSTOM pre/post needs n_chunks")
        C = int(n_chunks)
    if relay and pre is None:
        raise ValueError("relays need a CUSTOM or named collective")
    src, dst = topo.src, topo.dst
    threads = threads or min(len(seeds), os.cpu_count() or 1)

    def run(args):
        s, sig, a, b, allow = args
        return greedy(n, a, b, w, C, chunks_per_npu, s, sig, pre, post, record, literal, allow)

    rev = reverse_links(src, dst, w)
    need_rs = collective in ("RS", "AR", "REDUCE", "GATHER")
    only_rs = collective in ("RS", "REDUCE", "GATHER")
    rs_on_gt = need_rs and rev is None
    allow0 = _coll.relay_allow(n, src, dst, C, pre, post) if relay else None
    allow1 = _coll.relay_allow(n, dst, src, C, pre, post) if relay and rs_on_gt else None
    # searched jobs: the forward AG on G (sigma 0) unless only the G^T phase is used
    # (RS / REDUCE / GATHER on an asymmetric graph), and the AG on G^T (sigma 1) for the
    # RS phase of an asymmetric graph (R9).  V / D / M / E are summed over these jobs.
    jobs_ag = [] if (only_rs and rs_on_gt) else [(s, 0, src, dst, allow0) for s in seeds]
    jobs_rs = [(s, 1, dst, src, allow1) for s in seeds] if rs_on_gt else []
    with ThreadPoolExecutor(max_workers=threads) as ex:
        res = list(ex.map(run, jobs_ag + jobs_rs))
    ag = res[: len(jobs_ag)]
    rs = res[len(jobs_ag):] if jobs_rs else ag
    T_ag = np.array([r.T for r in ag], dtype=np.uint64)
    T_rs = np.array([r.T for r in rs], dtype=np.uint64)
    i_ag = int(np.argmin(T_ag)) if len(ag) else 0  # argmin returns the first (lowest index) minimum
    if not need_rs:  # AG, CUSTOM, BROADCAST, SCATTER
        win = ag[i_ag]
        return Synthesis(collective, win.T, canonical(win.sends) if record else win.sends, seeds[i_ag], seeds[i_ag],
                         win.T, 0, T_ag, ag, [])
    if rev is not None:
        # symmetric: RS_s = mirror(AG_s); T_AR(s) = 2 T_AG(s)
        t_ar = T_ag * np.uint64(2) if collective == "AR" else T_ag
        i_ag = i_rs = int(np.argmin(t_ar))
    else:
        # asymmetric: the RS and AG winners are chosen independently (T_AR = min T_RS + min T_AG);
        # the per-seed collective time is T_RS(s) + T_AG(s)
        i_rs = int(np.argmin(T_rs))
        t_ar = (T_rs + T_ag) if collective == "AR" else T_rs
    win_rs = rs[i_rs]
    T_RS = win_rs.T
    rs_sends = mirror(win_rs.sends, T_RS, src, dst, rev) if record else win_rs.sends[:0]
    if only_rs:
        return Synthesis(collective, T_RS, canonical(rs_sends), seeds[i_rs], seeds[i_rs], 0, T_RS, T_rs, ag, rs)
    win_ag = ag[i_ag]
    ag_sh = win_ag.sends.copy()
    ag_sh["t_start"] += np.uint64(T_RS)
    ag_sh["t_end"] += np.uint64(T_RS)
    allr = np.concatenate([rs_sends, ag_sh]) if record else ag_sh[:0]
    return Synthesis("AR", T_RS + win_ag.T, canonical(allr), seeds[i_ag], seeds[i_rs], win_ag.T, T_RS, t_ar, ag, rs)


def bits_from_sets(n_npus: int, n_chunks: int, sets: Dict[int, Sequence[int]]) -> np.ndarray:
    """Helper for CUSTOM pre/post: {npu: [chunks]} -> N x ceil(C/32) u32 words."""
    Wd = (n_chunks + 31) // 32
    out = np.zeros((n_npus, Wd), dtype=np.uint32)
    for x, cs in sets.items():
        for c in cs:
            out[x, c >> 5] |= np.uint32(1 << (c & 31))
    return out
