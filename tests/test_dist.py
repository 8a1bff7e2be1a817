"""Multi-process (world size 2 and 3, gloo, CPU) tests of the host logic of the multi-GPU
path: the library's ownership rule (include/zz.h zz_shard_columns, host
only) partitions the selected columns over the ranks with a pair never split, and the
columns each rank computes for its own share, gathered on rank 0, assemble the full result
bit for bit (column independence).  The per-rank solver here is the oracle
(tests may call it); on GPUs it is the collective zz_tgevc (tests/test_gpu.py covers that
path on one GPU through a one-rank communicator and zz_set_shard)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gen
import oracle
import paper_2003_04776_b200 as zz
from paper_2003_04776_b200 import dist as zdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, seed, frac, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    S0, T0, _ = gen.config(name, seed=seed)
    m = S0.shape[0]
    sub = np.diagonal(S0, -1).copy()
    sel = None
    if frac is not None:
        sel = (np.random.default_rng(seed).random(m) < frac).astype(np.int32)
    # the rank's share (library host logic), computed for its eigenvalue rows only
    cols = zdist.owned_columns(sub, m, world, rank, select=sel)
    rows = zdist.column_rows(sub, m, sel)[cols]
    sel_r = np.zeros(m, np.int32)
    sel_r[rows] = 1
    r = oracle.tgevc(S0, T0, select=sel_r) if len(cols) else {"X": np.zeros((m, 0)), "e": np.zeros(0, np.int32)}
    Xl = torch.from_numpy(np.ascontiguousarray(r["X"].T))        # (n_local, m)
    El = torch.from_numpy(r["e"].astype(np.int32))
    C = torch.from_numpy(cols.astype(np.int64))
    n = torch.tensor([len(cols)])
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n)
    if rank == 0:
        n_tot = int(sum(int(v) for v in ns))
        X = np.full((m, n_tot), np.nan, order="F")
        E = np.zeros(n_tot, np.int32)
        X[:, cols] = Xl.numpy().T
        E[cols] = El.numpy()
        for src in range(1, world):
            k = int(ns[src])
            if k == 0:
                continue
            bx = torch.empty((k, m), dtype=torch.float64)
            be = torch.empty(k, dtype=torch.int32)
            bc = torch.empty(k, dtype=torch.int64)
            dist.recv(bx, src)
            dist.recv(be, src)
            dist.recv(bc, src)
            X[:, bc.numpy()] = bx.numpy().T
            E[bc.numpy()] = be.numpy()
        q.put((X, E))
    elif len(cols):
        dist.send(Xl.contiguous(), 0)
        dist.send(El, 0)
        dist.send(C, 0)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,name,seed,frac", [(2, "C1", 3, None), (3, "C1", 4, None), (2, "C1", 5, 0.4)])
def test_ranks_assemble_bitwise(world, name, seed, frac):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, seed, frac, q)) for r in range(world)]
    for p in procs:
        p.start()
    X, E = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    S0, T0, _ = gen.config(name, seed=seed)
    sel = None if frac is None else (np.random.default_rng(seed).random(S0.shape[0]) < frac).astype(np.int32)
    ref = oracle.tgevc(S0, T0, select=sel)
    assert np.array_equal(X, ref["X"])
    assert np.array_equal(E, ref["e"])


@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_shard_columns_partition(P):
    S0, _, _ = gen.config("C2", seed=0)
    m = S0.shape[0]
    sub = np.diagonal(S0, -1).copy()
    first_row = np.zeros(m, int)
    for j, sz in zdist.block_layout(sub, m):
        first_row[j:j + sz] = j
    for sel in (None, (np.random.default_rng(P).random(m) < 0.3).astype(np.int32)):
        n = oracle.count_columns(S0, sel)
        rows = zdist.column_rows(sub, m, sel)
        assert len(rows) == n
        seen = np.zeros(n, int)
        for p in range(P):
            cols = zz.shard_columns(sub, m, P, p, select=sel)
            assert np.all(np.diff(cols) > 0)
            seen[cols] += 1
            # ownership by groups of 64 eigenvalue rows (first row of the block), cyclic
            for c in cols:
                assert (first_row[rows[c]] // 64) % P == p
        assert np.all(seen == 1)
    # argument errors
    lib = zz.load()
    assert lib.zz_shard_columns(-1, None, None, 1, 0, None) == -1
    assert lib.zz_shard_columns(4, sub.ctypes.data, None, 0, 0, None) == -4
    assert lib.zz_shard_columns(4, sub.ctypes.data, None, 2, 2, None) == -5
