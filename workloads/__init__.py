"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no cost quantization, no
matching, no RNG draws of the greedy).  It only emits graphs -- link arrays
(src, dst, alpha_ns, bw_bytes_per_ns) in a canonical link-id order -- plus the
per-config collective parameters (chunks per NPU, chunk bytes, seeds), shaped
like the paper's workloads (PAPER.md P:L107, P:L288-289,
P:L374).
"""
from .topologies import (  # noqa: F401
    Topology,
    Workload,
    uni_ring,
    bi_ring,
    path,
    fully_connected,
    mesh2d,
    torus,
    hypercube,
    ring_fc_switch,
    switch_hypercube_hybrid,
    random_strongly_connected,
    remove_undirected_links,
    is_strongly_connected,
    transpose,
    config,
    CONFIGS,
)
