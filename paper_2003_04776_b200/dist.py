"""Multi-GPU sharding (one process per GPU, torch.distributed for the plumbing).

The task graph of the method is a disjoint union of per-column subgraphs,
so eigenvector columns need no exchange during the computation.  Column blocks of width
`nb` are owned cyclically (block J -> rank J mod P, for triangular load balance); a complex
pair belongs to the block of its first column.  Each rank runs the full bottom-up wavefront
restricted to its own columns through the `select` argument of zz_tgevc, so the per-column
arithmetic is identical for any P and X is bitwise independent of P.

Collectives (NCCL on GPUs, gloo in the CPU tests): one broadcast of S and T from rank 0,
one gather of the computed columns to rank 0.
"""
import numpy as np


def block_layout(sub, m):
    """(start row, size) of the diagonal blocks from the subdiagonal S(j+1, j)."""
    out = []
    j = 0
    while j < m:
        two = j + 1 < m and sub[j] != 0.0
        out.append((j, 2 if two else 1))
        j += 2 if two else 1
    return out


def shard_select(sub, m, rank, world, nb=64):
    """int32 select mask of the eigenvalues owned by `rank` and the global output column
    indices of those columns (all eigenvectors computed; column index = row index)."""
    sel = np.zeros(m, np.int32)
    cols = []
    for j, sz in block_layout(sub, m):
        if (j // nb) % world == rank:
            sel[j:j + sz] = 1
            cols.extend(range(j, j + sz))
    return sel, np.asarray(cols, dtype=np.int64)


def tgevc_distributed(S, T, rank, world, compute, nb=64, group=None, sub=None):
    """All eigenvectors with column blocks sharded over `world` ranks.

    S, T: on rank 0 the pencil (column-major tensors on this rank's device); on the other
    ranks preallocated tensors of the same shape that receive the broadcast.
    compute(S, T, select) -> (X_local, e_local): the per-rank solver (zz.tgevc on GPUs).
    Returns (X, e) on rank 0 (m x m), (None, None) elsewhere."""
    import torch
    import torch.distributed as dist
    m = S.shape[0]
    # one broadcast of the pencil (S and T are stored column-major: broadcast the storage)
    dist.broadcast(S.t(), src=0, group=group)
    dist.broadcast(T.t(), src=0, group=group)
    if sub is None:
        sub = torch.diagonal(S, -1).cpu().numpy() if m > 1 else np.zeros(0)
    sel, cols = shard_select(sub, m, rank, world, nb)
    Xl, el = compute(S, T, sel)
    n_local = torch.tensor([Xl.shape[1]], dtype=torch.int64, device=S.device)
    sizes = [torch.zeros_like(n_local) for _ in range(world)]
    dist.all_gather(sizes, n_local, group=group)
    sizes = [int(s.item()) for s in sizes]
    buf_l = Xl.t().contiguous()           # (n_local, m) row-major == column-major X_local
    if rank == 0:
        X = torch.empty((m, m), dtype=S.dtype, device=S.device)         # row c = column c
        E = torch.empty(m, dtype=torch.int32, device=S.device)
        for r in range(world):
            if sizes[r] == 0:
                continue
            _, cols_r = shard_select(sub, m, r, world, nb)
            if r == 0:
                bx, be = buf_l, el
            else:
                bx = torch.empty((sizes[r], m), dtype=S.dtype, device=S.device)
                be = torch.empty(sizes[r], dtype=torch.int32, device=S.device)
                dist.recv(bx, src=r, group=group)
                dist.recv(be, src=r, group=group)
            idx = torch.as_tensor(cols_r, device=S.device)
            X.index_copy_(0, idx, bx)
            E.index_copy_(0, idx, be)
        return X.t(), E
    if sizes[rank] > 0:
        dist.send(buf_l, dst=0, group=group)
        dist.send(el.contiguous(), dst=0, group=group)
    return None, None
