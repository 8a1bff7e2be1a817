"""Multi-process (world_size 2, gloo, CPU) test of the N > 1 host logic of
paper_2003_04776_b200/dist.py: broadcast of S and T, cyclic column-block ownership through
`select`, gather and assembly on rank 0.  The per-rank solver is injected; here it is the
oracle (tests may call it), so the assembled X must equal the oracle's full X bitwise."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gen
import oracle
from paper_2003_04776_b200 import dist as zdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, seed, nb, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    S0, T0, _ = gen.config(name, seed=seed)
    m = S0.shape[0]
    if rank == 0:
        S = torch.from_numpy(np.ascontiguousarray(S0.T)).t()
        T = torch.from_numpy(np.ascontiguousarray(T0.T)).t()
    else:
        # NaN everywhere: the broadcast must deliver every entry the solve reads (the
        # upper part and the subdiagonal) and nothing below is read
        S = torch.full((m, m), float("nan"), dtype=torch.float64).t()
        T = torch.full((m, m), float("nan"), dtype=torch.float64).t()

    def compute(S_, T_, sel):
        r = oracle.tgevc(S_.numpy(), T_.numpy(), select=sel)
        X = torch.from_numpy(np.asfortranarray(r["X"]))
        return X, torch.from_numpy(r["e"].astype(np.int32))

    X, E = zdist.tgevc_distributed(S, T, rank, world, compute, nb=nb)
    if rank == 0:
        q.put((X.numpy().copy(), E.numpy().copy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("nb,world", [(8, 2), (32, 2), (8, 3)])
def test_two_rank_sharding_bitwise(nb, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, "C1", 3, nb, q)) for r in range(world)]
    for p in procs:
        p.start()
    X, E = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    S0, T0, _ = gen.config("C1", seed=3)
    ref = oracle.tgevc(S0, T0)
    assert np.array_equal(X, ref["X"])
    assert np.array_equal(E, ref["e"])


def test_upper_chunks_cover_the_columns():
    for m in (1, 2, 7, 96, 1000):
        ch = zdist.upper_chunks(m)
        assert ch[0][0] == 0 and ch[-1][1] == m
        assert all(a < b for a, b in ch) and all(ch[i][1] == ch[i + 1][0] for i in range(len(ch) - 1))


def test_shard_select_partitions_columns():
    S0, _, _ = gen.config("C2", seed=0)
    m = S0.shape[0]
    sub = np.diagonal(S0, -1)
    seen = np.zeros(m, int)
    for r in range(4):
        sel, cols = zdist.shard_select(sub, m, r, 4, nb=64)
        assert np.array_equal(np.flatnonzero(sel), cols)
        seen[cols] += 1
    assert np.all(seen == 1)
    # pairs are never split between ranks
    for j, sz in zdist.block_layout(sub, m):
        if sz == 2:
            owners = [r for r in range(4) if zdist.shard_select(sub, m, r, 4, 64)[0][j]]
            owners2 = [r for r in range(4) if zdist.shard_select(sub, m, r, 4, 64)[0][j + 1]]
            assert owners == owners2
            break
