"""Multi-GPU sharding (one process per GPU, torch.distributed for the plumbing).

The task graph of the method is a disjoint union of per-column subgraphs,
so eigenvector columns need no exchange during the computation.  Column blocks of width
`nb` are owned cyclically (block J -> rank J mod P, for triangular load balance); a complex
pair belongs to the block of its first column.  Each rank runs the full bottom-up wavefront
restricted to its own columns through the `select` argument of zz_tgevc, so the per-column
arithmetic is identical for any P and X is bitwise independent of P.

Collectives (NCCL on GPUs, gloo in the CPU tests): a broadcast of the upper trapezoid of S
and T from rank 0 (the solve never reads below the subdiagonal: half the bytes of the full
matrices), in column chunks of equal size packed into contiguous buffers, and one gather of
the computed columns to rank 0 with all receives posted at once (batched point-to-point).
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
    broadcast_upper(S, rank, group=group)
    broadcast_upper(T, rank, group=group)
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
        # every receive posted at once: the ranks' columns arrive concurrently
        bufs, ops = {}, []
        for r in range(1, world):
            if sizes[r] == 0:
                continue
            bx = torch.empty((sizes[r], m), dtype=S.dtype, device=S.device)
            be = torch.empty(sizes[r], dtype=torch.int32, device=S.device)
            bufs[r] = (bx, be)
            ops += [dist.P2POp(dist.irecv, bx, r, group=group), dist.P2POp(dist.irecv, be, r, group=group)]
        for w in (dist.batch_isend_irecv(ops) if ops else []):
            w.wait()
        for r in range(world):
            if sizes[r] == 0:
                continue
            _, cols_r = shard_select(sub, m, r, world, nb)
            bx, be = (buf_l, el) if r == 0 else bufs[r]
            idx = torch.as_tensor(cols_r, device=S.device)
            X.index_copy_(0, idx, bx)
            E.index_copy_(0, idx, be)
        return X.t(), E
    if sizes[rank] > 0:
        ops = [dist.P2POp(dist.isend, buf_l, 0, group=group), dist.P2POp(dist.isend, el.contiguous(), 0, group=group)]
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    return None, None


def upper_chunks(m, n_chunks=16):
    """Column chunks [c0, c1) of about equal upper-trapezoid size (column c needs rows
    0 .. c+1: the upper part and the subdiagonal)."""
    k = max(1, min(n_chunks, m))
    cuts = sorted(set([0, m] + [int(round(m * np.sqrt(i / k))) for i in range(1, k)]))
    return [(a, b) for a, b in zip(cuts[:-1], cuts[1:]) if b > a]


def broadcast_upper(A, rank, group=None, n_chunks=16):
    """Broadcast the upper trapezoid of the column-major m x m tensor A from rank 0: chunk
    [c0, c1) sends rows 0 .. min(c1 + 1, m) of its columns, packed contiguously.  Entries
    below the subdiagonal are not sent (never read by the solve)."""
    import torch
    import torch.distributed as dist
    m = A.shape[0]
    At = A.t()                       # row c of At = column c of A
    for c0, c1 in upper_chunks(m, n_chunks):
        r = min(c1 + 1, m)
        if rank == 0:
            buf = At[c0:c1, :r].contiguous()
        else:
            buf = torch.empty((c1 - c0, r), dtype=A.dtype, device=A.device)
        dist.broadcast(buf, src=0, group=group)
        if rank != 0:
            At[c0:c1, :r].copy_(buf)
