"""Python binding of libtacos.so (include/tacos.h): argument marshalling only.

Every step of the synthesis runs in the CUDA kernels behind the C ABI; this
module only converts numpy / torch buffers into pointers and back.  There is
no CPU fallback: if libtacos.so is missing, importing the synthesis entry
points raises; if no CUDA device is present, they raise TacosError(TACOS_E_CUDA).

Names follow the C ABI (tacos_load_topology, tacos_synthesize, tacos_eval, ...);
`Topology`, `synthesize`, `evaluate` and `Plan` are thin conveniences on top.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TACOS_LIB") or os.path.join(_HERE, "libtacos.so")  # TACOS_LIB: a tuning variant built by build.py --variant

TACOS_OK = 0
TACOS_E_INVALID_ARG = -1
TACOS_E_TOPOLOGY = -2
TACOS_E_UNREACHABLE = -3
TACOS_E_CUDA = -4
TACOS_E_NOMEM = -5
TACOS_E_OVERFLOW = -6
TACOS_E_VERIFY = -7
TACOS_E_NCCL = -8
TACOS_E_CAPACITY = -9

TACOS_ALL_GATHER = 0
TACOS_REDUCE_SCATTER = 1
TACOS_ALL_REDUCE = 2
TACOS_CUSTOM = 3
TACOS_BROADCAST = 4
TACOS_REDUCE = 5
TACOS_SCATTER = 6
TACOS_GATHER = 7
COLLECTIVES = {"AG": TACOS_ALL_GATHER, "RS": TACOS_REDUCE_SCATTER, "AR": TACOS_ALL_REDUCE, "CUSTOM": TACOS_CUSTOM,
               "BROADCAST": TACOS_BROADCAST, "REDUCE": TACOS_REDUCE, "SCATTER": TACOS_SCATTER, "GATHER": TACOS_GATHER}

TACOS_FLAG_NO_SCHEDULE = 1
TACOS_FLAG_KEEP_SEED_TIMES = 2
TACOS_FLAG_LITERAL = 4
TACOS_FLAG_RELAY = 8

VIOLATIONS = ("no_such_link", "wrong_duration", "link_overlap", "unheld_at_depart", "duplicate_delivery",
              "post_unmet", "phase_order", "not_maximal", "not_shorter_first")

SEND_DTYPE = np.dtype(
    [("chunk", "<u4"), ("src", "<u4"), ("dst", "<u4"), ("link", "<u4"), ("t_start", "<u8"), ("t_end", "<u8")]
)

KEY_SEED_BITS = 20


class tacos_send(ctypes.Structure):
    _fields_ = [("chunk", ctypes.c_uint32), ("src", ctypes.c_uint32), ("dst", ctypes.c_uint32),
                ("link", ctypes.c_uint32), ("t_start", ctypes.c_uint64), ("t_end", ctypes.c_uint64)]


class tacos_synth_params(ctypes.Structure):
    _fields_ = [("collective", ctypes.c_int32), ("chunks_per_npu", ctypes.c_uint32), ("chunk_bytes", ctypes.c_uint64),
                ("time_unit_ns", ctypes.c_uint32), ("n_seeds", ctypes.c_uint32), ("base_seed", ctypes.c_uint64),
                ("seed_offset", ctypes.c_uint32), ("n_chunks", ctypes.c_uint32),
                ("pre_bits", ctypes.POINTER(ctypes.c_uint32)), ("post_bits", ctypes.POINTER(ctypes.c_uint32)),
                ("flags", ctypes.c_uint32), ("root", ctypes.c_uint32), ("n_devices", ctypes.c_uint32)]


class tacos_result(ctypes.Structure):
    _fields_ = [("T", ctypes.c_uint64), ("T_ag", ctypes.c_uint64), ("T_rs", ctypes.c_uint64),
                ("seed", ctypes.c_uint64), ("rs_seed", ctypes.c_uint64), ("n_sends", ctypes.c_uint64),
                ("matches", ctypes.c_uint64), ("visits", ctypes.c_uint64), ("dest_events", ctypes.c_uint64),
                ("events", ctypes.c_uint64), ("status", ctypes.c_int32), ("winner_local", ctypes.c_uint32),
                ("best_key_ag", ctypes.c_uint64), ("best_key_rs", ctypes.c_uint64), ("cancelled", ctypes.c_uint64),
                ("live_visits", ctypes.c_uint64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class tacos_winner(ctypes.Structure):
    _fields_ = [("T", ctypes.c_uint64), ("T_ag", ctypes.c_uint64), ("T_rs", ctypes.c_uint64),
                ("seed_index_ag", ctypes.c_uint64), ("seed_index_rs", ctypes.c_uint64), ("local", ctypes.c_uint32),
                ("reserved", ctypes.c_uint32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_ if f != "reserved"}


class tacos_plan_info(ctypes.Structure):
    _fields_ = [("n_jobs", ctypes.c_uint32), ("ctas", ctypes.c_uint32), ("cluster", ctypes.c_uint32),
                ("threads", ctypes.c_uint32), ("smem_bytes", ctypes.c_uint32), ("rows_in_smem", ctypes.c_uint32),
                ("links_in_smem", ctypes.c_uint32), ("launches", ctypes.c_uint32), ("rows_bytes", ctypes.c_uint64),
                ("event_loop", ctypes.c_uint32), ("reserved", ctypes.c_uint32)]


class tacos_cont_report(ctypes.Structure):
    _fields_ = [("T_ns", ctypes.c_double), ("T_rs_ns", ctypes.c_double), ("max_link_busy_ns", ctypes.c_double),
                ("n_sends", ctypes.c_uint64)]


TACOS_BASELINE_RING, TACOS_BASELINE_DIRECT = 0, 1
BASELINES = {"ring": TACOS_BASELINE_RING, "direct": TACOS_BASELINE_DIRECT}


class tacos_dim_spec(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("n", ctypes.c_uint32), ("degree", ctypes.c_uint32),
                ("bidirectional", ctypes.c_uint32), ("alpha_ns", ctypes.c_uint32), ("bw", ctypes.c_uint32)]


TACOS_DIM_RING, TACOS_DIM_FC, TACOS_DIM_SWITCH, TACOS_DIM_PATH = 0, 1, 2, 3


class tacos_tenant(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("root", ctypes.c_uint32), ("k", ctypes.c_uint32)]
DIM_KINDS = {"ring": TACOS_DIM_RING, "fc": TACOS_DIM_FC, "switch": TACOS_DIM_SWITCH, "path": TACOS_DIM_PATH}


class tacos_eval_report(ctypes.Structure):
    _fields_ = [("T", ctypes.c_uint64), ("T_rs", ctypes.c_uint64), ("n_violations", ctypes.c_uint64),
                ("per_kind", ctypes.c_uint64 * len(VIOLATIONS)), ("first_kind", ctypes.c_int32), ("reserved", ctypes.c_uint32),
                ("first_index", ctypes.c_uint64)]


assert ctypes.sizeof(tacos_send) == 32

# every exported entry point declared in include/tacos.h: (restype, argtypes)
_VP = ctypes.c_void_p
_U32P = ctypes.POINTER(ctypes.c_uint32)
_I32P = ctypes.POINTER(ctypes.c_int32)
_U64P = ctypes.POINTER(ctypes.c_uint64)
SIGNATURES = {
    "tacos_load_topology": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, _I32P, _I32P, _U32P, _U32P, ctypes.POINTER(_VP)]),
    "tacos_free_topology": (None, [_VP]),
    "tacos_topology_num_npus": (ctypes.c_int32, [_VP]),
    "tacos_topology_num_links": (ctypes.c_int32, [_VP]),
    "tacos_topology_strongly_connected": (ctypes.c_int, [_VP]),
    "tacos_link_costs": (ctypes.c_int, [_VP, ctypes.c_uint64, ctypes.c_uint32, _U32P]),
    "tacos_is_symmetric": (ctypes.c_int, [_VP, ctypes.c_uint64, ctypes.c_uint32]),
    "tacos_synthesize": (ctypes.c_int, [_VP, ctypes.POINTER(tacos_synth_params), ctypes.POINTER(_VP)]),
    "tacos_synthesize_batch": (ctypes.c_int, [ctypes.POINTER(_VP), ctypes.c_uint32, ctypes.POINTER(tacos_synth_params), ctypes.POINTER(_VP)]),
    "tacos_synthesize_into": (ctypes.c_int, [_VP, ctypes.POINTER(tacos_synth_params), _VP, ctypes.c_uint64,
                                             ctypes.POINTER(tacos_result), _VP]),
    "tacos_max_sends": (ctypes.c_int, [_VP, ctypes.POINTER(tacos_synth_params), _U64P]),
    "tacos_schedule_num_sends": (ctypes.c_uint64, [_VP]),
    "tacos_schedule_sends": (_VP, [_VP]),
    "tacos_schedule_time": (ctypes.c_uint64, [_VP]),
    "tacos_schedule_seed": (ctypes.c_uint64, [_VP]),
    "tacos_schedule_result": (ctypes.POINTER(tacos_result), [_VP]),
    "tacos_schedule_seed_times": (_U64P, [_VP]),
    "tacos_free_schedule": (None, [_VP]),
    "tacos_plan_create": (ctypes.c_int, [_VP, ctypes.POINTER(tacos_synth_params), ctypes.POINTER(_VP)]),
    "tacos_plan_destroy": (None, [_VP]),
    "tacos_plan_search": (ctypes.c_int, [_VP, _VP]),
    "tacos_plan_best_keys": (_VP, [_VP]),
    "tacos_plan_emit": (ctypes.c_int, [_VP, _VP, ctypes.c_uint64, ctypes.POINTER(tacos_result), _VP]),
    "tacos_plan_seed_times_device": (_VP, [_VP, ctypes.POINTER(_VP)]),
    "tacos_plan_emit_async": (ctypes.c_int, [_VP, _VP, ctypes.c_uint64, _VP]),
    "tacos_plan_result": (ctypes.c_int, [_VP, ctypes.c_uint64, ctypes.POINTER(tacos_result), _VP]),
    "tacos_select_winner": (ctypes.c_int, [ctypes.POINTER(ctypes.c_uint64), ctypes.c_int32, ctypes.c_int,
                                           ctypes.c_uint32, ctypes.c_uint32, ctypes.POINTER(tacos_winner)]),
    "tacos_plan_last_launches": (ctypes.c_uint32, [_VP]),
    "tacos_plan_info_get": (ctypes.c_int, [_VP, ctypes.POINTER(tacos_plan_info)]),
    "tacos_plan_stats": (ctypes.c_int, [_VP, ctypes.POINTER(tacos_result), _VP]),
    "tacos_eval": (ctypes.c_int, [_VP, ctypes.POINTER(tacos_synth_params), _VP, ctypes.c_uint64,
                                  ctypes.POINTER(tacos_eval_report)]),
    "tacos_eval_continuous": (ctypes.c_int, [_VP, ctypes.POINTER(tacos_synth_params), _VP, ctypes.c_uint64,
                                             ctypes.POINTER(tacos_cont_report)]),
    "tacos_baseline": (ctypes.c_int, [_VP, ctypes.POINTER(tacos_synth_params), ctypes.c_int32, _VP, ctypes.c_uint64,
                                      _U64P]),
    "tacos_build_hierarchical": (ctypes.c_int, [ctypes.POINTER(tacos_dim_spec), ctypes.c_uint32, _I32P, _I32P, _I32P,
                                                _I32P, _U32P, _U32P, ctypes.c_int64]),
    "tacos_remove_npus": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, _I32P, _I32P, _U32P, _U32P, _I32P,
                                         ctypes.c_uint32, _I32P, _I32P, _I32P, _I32P, _U32P, _U32P, ctypes.c_int64,
                                         _I32P]),
    "tacos_comm_unique_id": (ctypes.c_int, [ctypes.POINTER(ctypes.c_uint8)]),
    "tacos_comm_init_rank": (ctypes.c_int, [ctypes.POINTER(ctypes.c_uint8), ctypes.c_int32, ctypes.c_int32,
                                            ctypes.POINTER(_VP)]),
    "tacos_comm_destroy": (None, [_VP]),
    "tacos_plan_allreduce_keys": (ctypes.c_int, [_VP, _VP, _VP]),
    "tacos_nccl_version": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int32)]),
    "tacos_multi_tenant": (ctypes.c_int, [ctypes.c_uint32, ctypes.POINTER(tacos_tenant), ctypes.c_uint32, _U32P,
                                          _U32P, _U32P, _U32P, ctypes.c_uint64]),
    "tacos_strerror": (ctypes.c_char_p, [ctypes.c_int]),
    "tacos_last_error": (ctypes.c_char_p, []),
    "tacos_abi_version": (ctypes.c_int, []),
    "tacos_philox_device": (ctypes.c_int, [_U32P, _U32P, _U32P]),
}

_lib = None


def load_library(path: str = LIB_PATH):
    """Load libtacos.so (built in-tree by paper_2304_05301_b200/build.py).
    Fails loudly: there is no fallback implementation."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise ImportError(f"libtacos.so not built at {path}; run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)  # AttributeError if a declared symbol is missing
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


class TacosError(RuntimeError):
    def __init__(self, code: int, where: str):
        lib = load_library()
        detail = lib.tacos_last_error().decode(errors="replace")
        super().__init__(f"{where}: {lib.tacos_strerror(code).decode()} ({code}): {detail}")
        self.code = code


def _check(rc: int, where: str):
    if rc != TACOS_OK:
        raise TacosError(rc, where)


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def _ptr(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


# --------------------------------------------------------------------------
# C ABI, same names
# --------------------------------------------------------------------------
def tacos_load_topology(n_npus: int, src, dst, alpha_ns, bw) -> ctypes.c_void_p:
    lib = load_library()
    s = np.ascontiguousarray(src, dtype=np.int32)
    d = np.ascontiguousarray(dst, dtype=np.int32)
    a = _u32(alpha_ns)
    b = _u32(bw)
    h = ctypes.c_void_p()
    _check(lib.tacos_load_topology(n_npus, s.shape[0], _ptr(s, ctypes.c_int32), _ptr(d, ctypes.c_int32),
                                   _ptr(a, ctypes.c_uint32), _ptr(b, ctypes.c_uint32), ctypes.byref(h)),
           "tacos_load_topology")
    return h


def tacos_free_topology(h):
    load_library().tacos_free_topology(h)


def make_params(collective="AR", chunks_per_npu=1, chunk_bytes=1 << 20, n_seeds=1, base_seed=0, seed_offset=0,
                time_unit_ns=1, flags=0, pre=None, post=None, n_chunks=0, root=0,
                n_devices=0) -> Tuple[tacos_synth_params, tuple]:
    """Build tacos_synth_params; returns (params, keepalive)."""
    p = tacos_synth_params()
    p.root = root
    p.n_devices = n_devices
    p.collective = COLLECTIVES[collective] if isinstance(collective, str) else int(collective)
    p.chunks_per_npu = chunks_per_npu
    p.chunk_bytes = chunk_bytes
    p.time_unit_ns = time_unit_ns
    p.n_seeds = n_seeds
    p.base_seed = base_seed & (2**64 - 1)
    p.seed_offset = seed_offset
    p.flags = flags
    keep = ()
    if pre is not None:
        pre_a = _u32(pre).ravel()
        post_a = _u32(post).ravel()
        p.pre_bits = _ptr(pre_a, ctypes.c_uint32)
        p.post_bits = _ptr(post_a, ctypes.c_uint32)
        p.n_chunks = n_chunks
        keep = (pre_a, post_a)
    return p, keep


def tacos_synthesize(topo_h, params: tacos_synth_params) -> ctypes.c_void_p:
    out = ctypes.c_void_p()
    _check(load_library().tacos_synthesize(topo_h, ctypes.byref(params), ctypes.byref(out)), "tacos_synthesize")
    return out


def tacos_synthesize_batch(topo_hs: Sequence, params: tacos_synth_params):
    n = len(topo_hs)
    arr = (ctypes.c_void_p * n)(*[t.value if isinstance(t, ctypes.c_void_p) else t for t in topo_hs])
    outs = (ctypes.c_void_p * n)()
    _check(load_library().tacos_synthesize_batch(arr, n, ctypes.byref(params), outs), "tacos_synthesize_batch")
    return [ctypes.c_void_p(o) for o in outs]


def tacos_schedule_sends(sched_h) -> np.ndarray:
    lib = load_library()
    n = lib.tacos_schedule_num_sends(sched_h)
    if n == 0:
        return np.zeros(0, dtype=SEND_DTYPE)
    ptr = lib.tacos_schedule_sends(sched_h)
    buf = (ctypes.c_char * (n * 32)).from_address(ptr)
    return np.frombuffer(buf, dtype=SEND_DTYPE, count=n).copy()


def tacos_schedule_result(sched_h) -> dict:
    return load_library().tacos_schedule_result(sched_h).contents.as_dict()


def tacos_schedule_seed_times(sched_h, n_seeds: int) -> Optional[np.ndarray]:
    p = load_library().tacos_schedule_seed_times(sched_h)
    if not p:
        return None
    return np.ctypeslib.as_array(p, shape=(n_seeds,)).copy()


def tacos_free_schedule(sched_h):
    load_library().tacos_free_schedule(sched_h)


def tacos_eval(topo_h, params: tacos_synth_params, sends: np.ndarray) -> dict:
    rep = tacos_eval_report()
    s = np.ascontiguousarray(sends, dtype=SEND_DTYPE)
    _check(load_library().tacos_eval(topo_h, ctypes.byref(params), s.ctypes.data, s.shape[0], ctypes.byref(rep)),
           "tacos_eval")
    out = {"T": rep.T, "T_rs": rep.T_rs, "n_violations": rep.n_violations, "first_kind": rep.first_kind,
           "first_index": rep.first_index}
    for i, k in enumerate(VIOLATIONS):
        out[k] = rep.per_kind[i]
    return out


NO_KEY = 0x7FFFFFFFFFFFFFFF


def make_key(T: int, seed_index: int) -> int:
    """Best-of-S key of one seed: (T << 20) | global seed index."""
    return (int(T) << KEY_SEED_BITS) | int(seed_index)


def tacos_select_winner(keys, collective, symmetric: bool, seed_offset: int, n_seeds: int) -> dict:
    k = (ctypes.c_uint64 * 2)(*[int(x) & (2**64 - 1) for x in keys])
    w = tacos_winner()
    c = COLLECTIVES[collective] if isinstance(collective, str) else int(collective)
    _check(load_library().tacos_select_winner(k, c, int(bool(symmetric)), seed_offset, n_seeds, ctypes.byref(w)),
           "tacos_select_winner")
    return w.as_dict()


def tacos_link_costs(topo_h, chunk_bytes: int, time_unit_ns: int = 1) -> np.ndarray:
    lib = load_library()
    n = lib.tacos_topology_num_links(topo_h)
    w = np.zeros(n, dtype=np.uint32)
    _check(lib.tacos_link_costs(topo_h, chunk_bytes, time_unit_ns, _ptr(w, ctypes.c_uint32)), "tacos_link_costs")
    return w


def tacos_philox_device(ctr, key):
    c = _u32(ctr)
    k = _u32(key)
    o = np.zeros(4, np.uint32)
    _check(load_library().tacos_philox_device(_ptr(c, ctypes.c_uint32), _ptr(k, ctypes.c_uint32),
                                              _ptr(o, ctypes.c_uint32)), "tacos_philox_device")
    return [int(x) for x in o]


# --------------------------------------------------------------------------
# conveniences
# --------------------------------------------------------------------------
class Topology:
    """Owns a tacos_topology handle."""

    def __init__(self, n_npus: int, src, dst, alpha_ns, bw):
        self.handle = tacos_load_topology(n_npus, src, dst, alpha_ns, bw)
        self.n_npus = n_npus
        self.n_links = int(np.asarray(src).shape[0])

    @classmethod
    def from_workload_topology(cls, t) -> "Topology":
        return cls(t.n_npus, t.src, t.dst, t.alpha_ns, t.bw)

    @property
    def strongly_connected(self) -> bool:
        return bool(load_library().tacos_topology_strongly_connected(self.handle))

    def link_costs(self, chunk_bytes: int, time_unit_ns: int = 1) -> np.ndarray:
        return tacos_link_costs(self.handle, chunk_bytes, time_unit_ns)

    def is_symmetric(self, chunk_bytes: int, time_unit_ns: int = 1) -> bool:
        return bool(load_library().tacos_is_symmetric(self.handle, chunk_bytes, time_unit_ns))

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and _lib is not None:
            _lib.tacos_free_topology(h)
            self.handle = None


@dataclass
class Schedule:
    sends: np.ndarray
    result: dict
    seed_times: Optional[np.ndarray] = None

    @property
    def T(self) -> int:
        return int(self.result["T"])


def synthesize(topo: Topology, collective="AR", chunks_per_npu=1, chunk_bytes=1 << 20, n_seeds=1, base_seed=0,
               time_unit_ns=1, keep_seed_times=False, no_schedule=False, pre=None, post=None,
               n_chunks=0, literal=False, relay=False, root=0, n_devices=0) -> Schedule:
    """tacos_synthesize.  collective: AG / RS / AR / CUSTOM (pre, post, n_chunks; relay=True
    for relays, R22) or the rooted BROADCAST / REDUCE / SCATTER / GATHER (root)."""
    flags = ((TACOS_FLAG_KEEP_SEED_TIMES if keep_seed_times else 0) | (TACOS_FLAG_NO_SCHEDULE if no_schedule else 0)
             | (TACOS_FLAG_LITERAL if literal else 0) | (TACOS_FLAG_RELAY if relay else 0))
    p, keep = make_params(collective, chunks_per_npu, chunk_bytes, n_seeds, base_seed, 0, time_unit_ns, flags, pre,
                          post, n_chunks, root, n_devices)
    h = tacos_synthesize(topo.handle, p)
    try:
        sends = tacos_schedule_sends(h)
        res = tacos_schedule_result(h)
        times = tacos_schedule_seed_times(h, n_seeds) if keep_seed_times else None
    finally:
        tacos_free_schedule(h)
    del keep
    return Schedule(sends, res, times)


def synthesize_batch(topos: Sequence[Topology], **kw) -> list:
    n_seeds = kw.get("n_seeds", 1)
    keep_times = kw.pop("keep_seed_times", False)
    flags = TACOS_FLAG_KEEP_SEED_TIMES if keep_times else 0
    p, keep = make_params(kw.get("collective", "AR"), kw.get("chunks_per_npu", 1), kw.get("chunk_bytes", 1 << 20),
                          n_seeds, kw.get("base_seed", 0), 0, kw.get("time_unit_ns", 1), flags,
                          n_devices=kw.get("n_devices", 0))
    hs = tacos_synthesize_batch([t.handle for t in topos], p)
    out = []
    for h in hs:
        try:
            out.append(Schedule(tacos_schedule_sends(h), tacos_schedule_result(h),
                                tacos_schedule_seed_times(h, n_seeds) if keep_times else None))
        finally:
            tacos_free_schedule(h)
    return out


def max_sends(topo: Topology, params: tacos_synth_params) -> int:
    n = ctypes.c_uint64(0)
    _check(load_library().tacos_max_sends(topo.handle, ctypes.byref(params), ctypes.byref(n)), "tacos_max_sends")
    return int(n.value)


def synthesize_into(topo: Topology, params: tacos_synth_params, sends_ptr: int, capacity: int, stream: int = 0):
    """tacos_synthesize_into: sends_ptr is a host (pinned) or device address."""
    res = tacos_result()
    _check(load_library().tacos_synthesize_into(topo.handle, ctypes.byref(params), ctypes.c_void_p(sends_ptr),
                                                capacity, ctypes.byref(res), ctypes.c_void_p(stream)),
           "tacos_synthesize_into")
    return res.as_dict()


def evaluate(topo: Topology, sends: np.ndarray, collective="AR", chunks_per_npu=1, chunk_bytes=1 << 20,
             time_unit_ns=1, pre=None, post=None, n_chunks=0, root=0, literal=False, relay=False) -> dict:
    """tacos_eval.  literal / relay name the variant that produced the schedule (the
    greedy-rule checks apply to link-first searches without relays only)."""
    flags = (TACOS_FLAG_LITERAL if literal else 0) | (TACOS_FLAG_RELAY if relay else 0)
    p, keep = make_params(collective, chunks_per_npu, chunk_bytes, 1, 0, 0, time_unit_ns, flags, pre, post, n_chunks,
                          root)
    return tacos_eval(topo.handle, p, sends)


class _CudaArray:
    """__cuda_array_interface__ view of library-owned device memory."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"data": (ptr, False), "shape": tuple(shape), "typestr": typestr,
                                         "version": 3, "strides": None}


class Plan:
    """Device-resident plan (tacos_plan_*): search on a stream, all-reduce the
    best keys across ranks (caller), emit on the owning rank."""

    def __init__(self, topo: Topology, collective="AR", chunks_per_npu=1, chunk_bytes=1 << 20, n_seeds=1,
                 base_seed=0, seed_offset=0, time_unit_ns=1, no_schedule=False, literal=False, root=0,
                 pre=None, post=None, n_chunks=0, relay=False):
        self.topo = topo
        flags = ((TACOS_FLAG_NO_SCHEDULE if no_schedule else 0) | (TACOS_FLAG_LITERAL if literal else 0)
                 | (TACOS_FLAG_RELAY if relay else 0))
        self.params, self._keep = make_params(collective, chunks_per_npu, chunk_bytes, n_seeds, base_seed, seed_offset,
                                              time_unit_ns, flags, pre, post, n_chunks, root)
        h = ctypes.c_void_p()
        _check(load_library().tacos_plan_create(topo.handle, ctypes.byref(self.params), ctypes.byref(h)),
               "tacos_plan_create")
        self.handle = h
        self.n_sends = max_sends(topo, self.params)

    def search(self, stream: int = 0):
        _check(load_library().tacos_plan_search(self.handle, ctypes.c_void_p(stream)), "tacos_plan_search")

    def allreduce_keys(self, comm: "Comm", stream: int = 0):
        """tacos_plan_allreduce_keys: the cross-rank MIN of the best keys over NCCL."""
        _check(load_library().tacos_plan_allreduce_keys(self.handle, comm.handle, ctypes.c_void_p(stream)),
               "tacos_plan_allreduce_keys")

    def best_keys_ptr(self) -> int:
        return int(load_library().tacos_plan_best_keys(self.handle))

    def best_keys_tensor(self):
        """torch int64[2] aliasing the plan's device keys (for dist.all_reduce MIN)."""
        import torch

        return torch.as_tensor(_CudaArray(self.best_keys_ptr(), (2,), "<i8"), device="cuda")

    def emit(self, sends_ptr: int, capacity: int, stream: int = 0) -> dict:
        res = tacos_result()
        _check(load_library().tacos_plan_emit(self.handle, ctypes.c_void_p(sends_ptr), capacity, ctypes.byref(res),
                                              ctypes.c_void_p(stream)), "tacos_plan_emit")
        return res.as_dict()

    def emit_async(self, sends_ptr: int, capacity: int, stream: int = 0) -> bool:
        """tacos_plan_emit_async; False when this plan needs tacos_plan_emit instead."""
        rc = load_library().tacos_plan_emit_async(self.handle, ctypes.c_void_p(sends_ptr), capacity,
                                                   ctypes.c_void_p(stream))
        if rc == TACOS_E_INVALID_ARG:
            return False
        _check(rc, "tacos_plan_emit_async")
        return True

    def result(self, capacity: int, stream: int = 0) -> dict:
        res = tacos_result()
        _check(load_library().tacos_plan_result(self.handle, capacity, ctypes.byref(res), ctypes.c_void_p(stream)),
               "tacos_plan_result")
        return res.as_dict()

    def stats(self, stream: int = 0) -> dict:
        res = tacos_result()
        _check(load_library().tacos_plan_stats(self.handle, ctypes.byref(res), ctypes.c_void_p(stream)),
               "tacos_plan_stats")
        return res.as_dict()

    def info(self) -> dict:
        inf = tacos_plan_info()
        _check(load_library().tacos_plan_info_get(self.handle, ctypes.byref(inf)), "tacos_plan_info_get")
        return {f: getattr(inf, f) for f, _ in inf._fields_}

    def last_launches(self) -> int:
        return int(load_library().tacos_plan_last_launches(self.handle))

    def seed_times_ptr(self) -> int:
        rs = ctypes.c_void_p()
        return int(load_library().tacos_plan_seed_times_device(self.handle, ctypes.byref(rs)) or 0)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and _lib is not None:
            _lib.tacos_plan_destroy(h)
            self.handle = None


COMM_ID_BYTES = 128


def comm_unique_id() -> bytes:
    """tacos_comm_unique_id (rank 0), 128 bytes to ship to the other ranks."""
    buf = (ctypes.c_uint8 * COMM_ID_BYTES)()
    _check(load_library().tacos_comm_unique_id(buf), "tacos_comm_unique_id")
    return bytes(buf)


def nccl_version() -> int:
    v = ctypes.c_int32()
    _check(load_library().tacos_nccl_version(ctypes.byref(v)), "tacos_nccl_version")
    return int(v.value)


class Comm:
    """tacos_comm: one rank of a multi-process job, on the current CUDA device."""

    def __init__(self, unique_id: bytes, n_ranks: int, rank: int):
        buf = (ctypes.c_uint8 * COMM_ID_BYTES).from_buffer_copy(unique_id)
        h = ctypes.c_void_p()
        _check(load_library().tacos_comm_init_rank(buf, n_ranks, rank, ctypes.byref(h)), "tacos_comm_init_rank")
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and _lib is not None:
            _lib.tacos_comm_destroy(h)
            self.handle = None


def sends_from_bytes(buf: np.ndarray) -> np.ndarray:
    return np.frombuffer(np.ascontiguousarray(buf).tobytes(), dtype=SEND_DTYPE)


# --------------------------------------------------------------------------
# topology front-end (f4)
# --------------------------------------------------------------------------
def tacos_build_hierarchical(dims):
    """dims: list of dicts {kind: ring|fc|switch|path, n, degree=1, bidirectional=0,
    alpha_ns, bw}.  Returns (n_npus, src, dst, alpha_ns, bw) numpy arrays."""
    lib = load_library()
    arr = (tacos_dim_spec * len(dims))()
    for a, d in zip(arr, dims):
        a.kind = DIM_KINDS[d["kind"]] if isinstance(d["kind"], str) else int(d["kind"])
        a.n = d["n"]
        a.degree = d.get("degree", 1)
        a.bidirectional = int(d.get("bidirectional", 0))
        a.alpha_ns = d.get("alpha_ns", 500)
        a.bw = d["bw"]
    n = ctypes.c_int32()
    m = ctypes.c_int32()
    _check(lib.tacos_build_hierarchical(arr, len(dims), ctypes.byref(n), ctypes.byref(m), None, None, None, None, 0),
           "tacos_build_hierarchical")
    L = m.value
    src = np.zeros(L, np.int32)
    dst = np.zeros(L, np.int32)
    al = np.zeros(L, np.uint32)
    bw = np.zeros(L, np.uint32)
    _check(lib.tacos_build_hierarchical(arr, len(dims), ctypes.byref(n), ctypes.byref(m), _ptr(src, ctypes.c_int32),
                                        _ptr(dst, ctypes.c_int32), _ptr(al, ctypes.c_uint32), _ptr(bw, ctypes.c_uint32),
                                        L), "tacos_build_hierarchical")
    return n.value, src, dst, al, bw


def tacos_remove_npus(n_npus, src, dst, alpha_ns, bw, removed):
    lib = load_library()
    s_ = np.ascontiguousarray(src, np.int32)
    d_ = np.ascontiguousarray(dst, np.int32)
    a_ = _u32(alpha_ns)
    b_ = _u32(bw)
    r_ = np.ascontiguousarray(removed, np.int32)
    L = s_.shape[0]
    n2 = ctypes.c_int32()
    m2 = ctypes.c_int32()
    os_ = np.zeros(max(L, 1), np.int32)
    od_ = np.zeros(max(L, 1), np.int32)
    oa_ = np.zeros(max(L, 1), np.uint32)
    ob_ = np.zeros(max(L, 1), np.uint32)
    oid = np.zeros(max(n_npus, 1), np.int32)
    _check(lib.tacos_remove_npus(n_npus, L, _ptr(s_, ctypes.c_int32), _ptr(d_, ctypes.c_int32), _ptr(a_, ctypes.c_uint32),
                                 _ptr(b_, ctypes.c_uint32), _ptr(r_, ctypes.c_int32), r_.shape[0], ctypes.byref(n2),
                                 ctypes.byref(m2), _ptr(os_, ctypes.c_int32), _ptr(od_, ctypes.c_int32),
                                 _ptr(oa_, ctypes.c_uint32), _ptr(ob_, ctypes.c_uint32), max(L, n_npus),
                                 _ptr(oid, ctypes.c_int32)), "tacos_remove_npus")
    k = m2.value
    return n2.value, os_[:k].copy(), od_[:k].copy(), oa_[:k].copy(), ob_[:k].copy(), oid[:n2.value].copy()


# --------------------------------------------------------------------------
# continuous-time evaluation and baselines (f3)
# --------------------------------------------------------------------------
def evaluate_continuous(topo: Topology, sends: np.ndarray, collective="AR", chunks_per_npu=1, chunk_bytes=1 << 20,
                        pre=None, post=None, n_chunks=0, root=0) -> dict:
    p, keep = make_params(collective, chunks_per_npu, chunk_bytes, 1, 0, 0, 1, 0, pre, post, n_chunks, root)
    rep = tacos_cont_report()
    s_ = np.ascontiguousarray(sends, dtype=SEND_DTYPE)
    _check(load_library().tacos_eval_continuous(topo.handle, ctypes.byref(p), s_.ctypes.data, s_.shape[0],
                                                ctypes.byref(rep)), "tacos_eval_continuous")
    return {"T_ns": rep.T_ns, "T_rs_ns": rep.T_rs_ns, "max_link_busy_ns": rep.max_link_busy_ns, "n_sends": rep.n_sends}


def baseline(topo: Topology, algorithm="ring", collective="AR", chunks_per_npu=1, chunk_bytes=1 << 20) -> np.ndarray:
    p, keep = make_params(collective, chunks_per_npu, chunk_bytes, 1)
    lib = load_library()
    n = ctypes.c_uint64()
    alg = BASELINES[algorithm] if isinstance(algorithm, str) else int(algorithm)
    _check(lib.tacos_baseline(topo.handle, ctypes.byref(p), alg, None, 0, ctypes.byref(n)), "tacos_baseline")
    out = np.zeros(max(n.value, 1), dtype=SEND_DTYPE)
    _check(lib.tacos_baseline(topo.handle, ctypes.byref(p), alg, out.ctypes.data, n.value, ctypes.byref(n)),
           "tacos_baseline")
    return out[: n.value]


# --------------------------------------------------------------------------
# multi-tenant collectives (Table VI)
# --------------------------------------------------------------------------
def multi_tenant(n_npus: int, tenants) -> Tuple[int, np.ndarray, np.ndarray, list]:
    """tacos_multi_tenant: merge concurrent tenants (kind, root, k) -- kind AG (root
    unused), BROADCAST, SCATTER, GATHER or REDUCE -- into one CUSTOM pre/postcondition
    over disjoint chunk ranges, to be synthesized with relay=True (reading R23: a Reduce
    tenant is scheduled as the Gather of its N partial chunks).  Returns (C, pre, post,
    first chunk id of each tenant); pre/post are N x ceil(C/32) uint32 rows."""
    lib = load_library()
    arr = (tacos_tenant * len(tenants))()
    for a, (kind, root, k) in zip(arr, tenants):
        if kind not in ("AG", "BROADCAST", "SCATTER", "GATHER", "REDUCE"):
            raise ValueError(f"unknown tenant kind {kind}")
        a.kind = COLLECTIVES[kind]
        a.root = int(root)
        a.k = int(k)
    C = ctypes.c_uint32()
    _check(lib.tacos_multi_tenant(n_npus, arr, len(tenants), ctypes.byref(C), None, None, None, 0),
           "tacos_multi_tenant")
    words = (C.value + 31) // 32
    pre = np.zeros((n_npus, words), np.uint32)
    post = np.zeros((n_npus, words), np.uint32)
    first = np.zeros(len(tenants), np.uint32)
    _check(lib.tacos_multi_tenant(n_npus, arr, len(tenants), ctypes.byref(C), _ptr(pre, ctypes.c_uint32),
                                  _ptr(post, ctypes.c_uint32), _ptr(first, ctypes.c_uint32), pre.size),
           "tacos_multi_tenant")
    return int(C.value), pre, post, [int(x) for x in first]
