"""Several GPUs ("initiating multiple independent search
instances concurrently and choose the best"): the library's own seed sharding
(tacos_synth_params.n_devices: one host thread, stream and plan per device, one
ncclAllReduce MIN of the two best keys) and its multi-process communicator
(tacos_comm_*, tacos_plan_allreduce_keys) against the CPU oracle over the union
of the seeds.  Needs >= 2 visible GPUs (gpurun --gpus 2 / 4); skipped otherwise."""
import hashlib
import os

import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T():
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    from paper_2304_05301_b200 import build

    build.build()
    import paper_2304_05301_b200 as T

    T.load_library()
    return T


def _check(syn, sch, coll):
    from test_gpu_parity import assert_parity

    assert_parity(syn, sch, coll)


@pytest.mark.parametrize("devs", [2, 0xFFFFFFFF])
def test_sharded_seeds_equal_oracle_config2(T, devs):
    wl = W.config(2)
    syn = oracle.synthesize(wl.topo, 4, 1 << 20, "AR", list(range(64)))
    t = T.Topology.from_workload_topology(wl.topo)
    sch = T.synthesize(t, "AR", 4, 1 << 20, 64, keep_seed_times=True, n_devices=devs)
    _check(syn, sch, "AR")


def test_sharded_seeds_equal_oracle_config3(T):
    wl = W.config(3)
    syn = oracle.synthesize(wl.topo, 1, 1 << 20, "AR", list(range(64)))
    t = T.Topology.from_workload_topology(wl.topo)
    sch = T.synthesize(t, "AR", 1, 1 << 20, 64, keep_seed_times=True, n_devices=2)
    _check(syn, sch, "AR")


@pytest.mark.parametrize("coll", ["AR", "RS", "AG"])
def test_sharded_asymmetric_winners(T, coll):
    """Asymmetric graph: the RS phase (G^T search) and the AG phase may be won by seeds
    on different devices; each owner writes its half."""
    topo = W.ring_fc_switch(2, 4, 64, 200, 100, 50)
    syn = oracle.synthesize(topo, 1, 1 << 20, coll, list(range(12)))
    t = T.Topology.from_workload_topology(topo)
    sch = T.synthesize(t, coll, 1, 1 << 20, 12, keep_seed_times=True, n_devices=3 if _ndev() >= 3 else 2)
    _check(syn, sch, coll)


def _ndev():
    import torch

    return torch.cuda.device_count()


def test_sharded_rooted_relay_collective(T):
    topo = W.mesh2d(6, 6)
    syn = oracle.synthesize(topo, 1, 1 << 20, "GATHER", list(range(8)), root=17)
    t = T.Topology.from_workload_topology(topo)
    sch = T.synthesize(t, "GATHER", 1, 1 << 20, 8, keep_seed_times=True, n_devices=2, root=17)
    _check(syn, sch, "GATHER")


def test_batch_topologies_dealt_to_devices(T):
    topos = [W.config(5).topo, W.torus([8, 8]), W.mesh2d(8, 8, 200, 100), W.torus([4, 4, 4])]
    ts = [T.Topology.from_workload_topology(x) for x in topos]
    out = T.synthesize_batch(ts, collective="AR", chunks_per_npu=1, chunk_bytes=1 << 20, n_seeds=8,
                             keep_seed_times=True, n_devices=2)
    for x, b in zip(topos, out):
        _check(oracle.synthesize(x, 1, 1 << 20, "AR", list(range(8))), b, "AR")


def test_synthesize_into_device_buffer_sharded(T):
    import torch

    wl = W.config(3)
    t = T.Topology.from_workload_topology(wl.topo)
    p, keep = T.make_params("AR", 1, 1 << 20, 16, n_devices=2)
    n = T.max_sends(t, p)
    dev = torch.zeros(n * 32, dtype=torch.uint8, device="cuda:0")
    r = T.synthesize_into(t, p, dev.data_ptr(), n)
    syn = oracle.synthesize(wl.topo, 1, 1 << 20, "AR", list(range(16)))
    assert r["T"] == syn.T and r["n_sends"] == n and r["seed"] == syn.seed
    assert dev.cpu().numpy().tobytes() == syn.sends.tobytes()


def _rank(rank, world, q_id, q_out, S):
    import torch

    import paper_2304_05301_b200 as T

    torch.cuda.set_device(rank)
    T.load_library()
    if rank == 0:
        uid = T.comm_unique_id()
        for _ in range(world - 1):
            q_id.put(uid)
    else:
        uid = q_id.get(timeout=120)
    comm = T.Comm(uid, world, rank)
    wl = W.config(2)
    t = T.Topology.from_workload_topology(wl.topo)
    plan = T.Plan(t, "AR", 4, 1 << 20, S, 0, rank * S)
    st = torch.cuda.current_stream().cuda_stream
    plan.search(st)
    plan.allreduce_keys(comm, st)
    out = torch.zeros(plan.n_sends * 32, dtype=torch.uint8, device="cuda")
    res = plan.emit(out.data_ptr(), plan.n_sends, st)
    torch.cuda.synchronize()
    blob = out.cpu().numpy().tobytes() if res["winner_local"] else b""
    q_out.put((rank, res["T"], res["seed"], res["winner_local"], blob))


def test_multiprocess_comm_selects_global_winner(T):
    """One process per GPU (the torchrun shape): rank 0's NCCL id is shipped through a
    queue (no torch.distributed), each rank searches its seed block, the library's
    ncclAllReduce MIN picks the global winner, its owner emits the oracle's schedule."""
    import torch.multiprocessing as mp

    world, S = 2, 16
    ctx = mp.get_context("spawn")
    q_id, q_out = ctx.Queue(), ctx.Queue()
    procs = [ctx.Process(target=_rank, args=(r, world, q_id, q_out, S)) for r in range(world)]
    for p in procs:
        p.start()
    got = sorted([q_out.get(timeout=600) for _ in range(world)])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    syn = oracle.synthesize(W.config(2).topo, 4, 1 << 20, "AR", list(range(world * S)))
    assert all(g[1] == syn.T and g[2] == syn.seed for g in got)
    owners = [g for g in got if g[3]]
    assert len(owners) == 1 and owners[0][3] == 3
    assert owners[0][4] == syn.sends.tobytes()
