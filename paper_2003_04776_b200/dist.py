"""Multi-GPU helpers (one process per GPU; torch.distributed is plumbing only).

The method's task graph is a disjoint union of per-column-block subgraphs, so
eigenvector columns need no exchange during the computation.  The data
path lives in the C library (include/zz.h): zz_init(device, nranks, rank, id) creates an NCCL
communicator; the collective zz_tgevc then broadcasts the upper panels of S and T from rank 0
in the order the wavefront consumes them (overlapped with the solve), every rank solves the
eigenvalue blocks it owns (groups of 64 rows, cyclic over the ranks: zz_shard_columns), and
the finished columns (rows 0 .. r_c only) are gathered into rank 0's X.  This module only
exchanges the 128-byte NCCL id through torch.distributed and calls the library.
"""
import numpy as np

import paper_2003_04776_b200 as zz


def init(rank, world, device, group=None):
    """Create the library's multi-rank context on `device` (collective over `group`)."""
    return zz.init_distributed(rank, world, device=device, group=group)


def owned_columns(sub, m, world, rank, select=None):
    """Global output columns owned by `rank` (the library's ownership rule)."""
    return zz.shard_columns(sub, m, world, rank, select=select)


def block_layout(sub, m):
    """(start row, size) of the diagonal blocks from the subdiagonal S(j+1, j)."""
    out = []
    j = 0
    while j < m:
        two = j + 1 < m and sub[j] != 0.0
        out.append((j, 2 if two else 1))
        j += 2 if two else 1
    return out


def column_rows(sub, m, select=None):
    """eigenvalue row of every output column (block order; a pair's columns -> its rows)"""
    rows = []
    for j, sz in block_layout(sub, m):
        if select is None or select[j] or (sz == 2 and select[j + 1]):
            rows.extend(range(j, j + sz))
    return np.asarray(rows, dtype=np.int64)
