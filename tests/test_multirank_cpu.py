"""Multi-rank host logic on CPU (gloo, world_size 2): seed sharding, the one
exchange step (MIN all-reduce of the two best-of-S keys) and the
winner decode of the C ABI (tacos_select_winner).  Per-seed finish times come
from the oracle here (no GPU); on B200 the same keys come from
tacos_plan_search and the all-reduce runs over NCCL (bench.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import workloads as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case(name):
    if name == "sym":
        return W.torus([4, 4]), 2
    return W.random_strongly_connected(7, 16, 3, bws=(25, 100), alphas=(0, 500)), 1


def _worker(rank, world, port, name, S, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2304_05301_b200 as T

        topo, k = _case(name)
        seeds = list(range(rank * S, rank * S + S))
        syn = oracle.synthesize(topo, k, 1 << 20, "AR", seeds, threads=1)
        key_ag = min(T.make_key(g.T, s) for g, s in zip(syn.ag, seeds))
        key_rs = min(T.make_key(g.T, s) for g, s in zip(syn.rs, seeds))
        sym = syn.rs is syn.ag
        keys = torch.tensor([key_ag, key_rs if not sym else key_ag], dtype=torch.int64)
        dist.all_reduce(keys, op=dist.ReduceOp.MIN)
        win = T.tacos_select_winner(keys.tolist(), "AR", sym, rank * S, S)
        q.put((rank, win, sym))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["sym", "asym"])
def test_two_rank_selection_matches_single_process(name):
    from paper_2304_05301_b200 import build

    build.build()
    import paper_2304_05301_b200 as T

    S, world = 4, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, S, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got.sort(key=lambda x: x[0])
    topo, k = _case(name)
    ref = oracle.synthesize(topo, k, 1 << 20, "AR", list(range(world * S)))
    wins = [g[1] for g in got]
    # every rank decodes the same global winner
    for w in wins:
        assert w["T"] == ref.T and w["T_ag"] == ref.T_ag and w["T_rs"] == ref.T_rs
        assert w["seed_index_ag"] == ref.seed and w["seed_index_rs"] == ref.rs_seed
    # each phase is emitted by exactly one rank
    for bit in (1, 2):
        assert sum(1 for w in wins if w["local"] & bit) == 1
    assert got[0][2] == (name == "sym")


def test_select_winner_edge_cases():
    from paper_2304_05301_b200 import build

    build.build()
    import paper_2304_05301_b200 as T

    with pytest.raises(T.TacosError) as e:
        T.tacos_select_winner([T.NO_KEY, T.NO_KEY], "AG", True, 0, 4)
    assert e.value.code == T.TACOS_E_UNREACHABLE
    with pytest.raises(T.TacosError) as e:
        T.tacos_select_winner([T.make_key(1 << 40, 0), 0], "AG", True, 0, 4)
    assert e.value.code == T.TACOS_E_OVERFLOW
    w = T.tacos_select_winner([T.make_key(100, 5), T.make_key(70, 2)], "AR", False, 4, 4)
    assert (w["T"], w["T_ag"], w["T_rs"], w["seed_index_ag"], w["seed_index_rs"], w["local"]) == (170, 100, 70, 5, 2, 1)
    w = T.tacos_select_winner([T.make_key(100, 5), T.make_key(70, 2)], "AR", True, 4, 4)
    assert (w["T"], w["seed_index_rs"], w["local"]) == (200, 5, 3)
    w = T.tacos_select_winner([T.make_key(100, 5), T.make_key(70, 2)], "RS", False, 0, 4)
    assert (w["T"], w["T_ag"], w["seed_index_rs"], w["local"]) == (70, 0, 2, 2)
