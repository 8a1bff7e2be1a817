"""paper_2003_04776_b200 -- B200-native robust generalized eigenvectors of a real Schur pencil.

Thin ctypes binding of the C ABI in include/zz.h (argument marshalling only; every step of
the computation runs in the CUDA kernels of csrc/).  PyTorch is used for device memory and
streams.  There is no CPU fallback: without the built library or a CUDA device every call
raises.

Method: Kjelgaard Mikkelsen & Myllykoski, "Parallel Robust Computation of Generalized
Eigenvectors of Matrix Pencils": solve S V D - T V B = 0 by the
robust blocked back-substitution of Algorithm 1 with augmented matrices
and int32 power-of-two scaling exponents.
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libzz.so")
_lib = None

STATUS = {
    0: "success",
    -100: "CUDA error",
    -102: "out of device memory",
    -103: "no context",
    -104: "non-finite entry in a diagonal block",
    -105: "overlapping 2x2 blocks",
    -106: "unsupported tile size",
    -107: "a diagonal entry of T is not real (zz_ztgevc)",
    -101: "NCCL error",
    -108: "shard emulation not allowed here",
}

EXPORTS = ["zz_get_unique_id", "zz_init", "zz_set_shard", "zz_shard_columns", "zz_set_stream", "zz_set_tile", "zz_set_graphs", "zz_set_diag_team", "zz_set_timing", "zz_set_fusion", "zz_set_lookahead", "zz_tgevc", "zz_tgevc_host", "zz_tgevc_back", "zz_tgevc_left", "zz_ztgevc",
           "zz_count_columns", "zz_partition", "zz_last_info", "zz_finalize", "zz_status_string"]


class ZZError(RuntimeError):
    def __init__(self, status, what=""):
        self.status = status
        msg = STATUS.get(status, "2x2 block with real eigenvalues at row %d" % status if status > 0
                         else "invalid argument %d" % -status)
        super().__init__("%s: status %d (%s)" % (what or "zz", status, msg))


class Info(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int), ("n_sel", ctypes.c_int), ("mb", ctypes.c_int),
                ("n_tiles", ctypes.c_int), ("n_scaled", ctypes.c_int), ("min_exp", ctypes.c_int),
                ("n_indefinite", ctypes.c_int), ("prescaled", ctypes.c_int),
                ("update_launches", ctypes.c_int), ("total_launches", ctypes.c_int),
                ("fused_pairs", ctypes.c_int), ("lookahead_redo", ctypes.c_int),
                ("ms_setup", ctypes.c_double), ("ms_steps", ctypes.c_double),
                ("ms_normalize", ctypes.c_double), ("ms_update", ctypes.c_double),
                ("ms_back", ctypes.c_double),
                ("d_logmax", ctypes.c_void_p), ("d_a", ctypes.c_void_p), ("d_b", ctypes.c_void_p),
                ("d_beta", ctypes.c_void_p)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_cudart_lib = None


def _d2h(ptr, nbytes):
    """copy `nbytes` of device memory at `ptr` to a new host bytes buffer (cudaMemcpy)"""
    global _cudart_lib
    if _cudart_lib is None:
        import glob
        cands = []
        try:
            import nvidia.cuda_runtime as cr
            for d in cr.__path__:
                cands += sorted(glob.glob(os.path.join(d, "lib", "libcudart.so*")))
        except Exception:
            pass
        cands += ["libcudart.so.12", "libcudart.so"]
        for c in cands:
            try:
                _cudart_lib = ctypes.CDLL(c)
                break
            except OSError:
                continue
        if _cudart_lib is None:
            raise ImportError("libcudart not found")
        _cudart_lib.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
        _cudart_lib.cudaMemcpy.restype = ctypes.c_int
    buf = ctypes.create_string_buffer(max(int(nbytes), 1))
    if nbytes:
        st = _cudart_lib.cudaMemcpy(buf, ctypes.c_void_p(ptr), int(nbytes), 2)
        if st != 0:
            raise RuntimeError("cudaMemcpy (device views) failed: %d" % st)
    return buf.raw[:nbytes]


def library_path():
    return _SO


def load(build_if_missing=True):
    """Load libzz.so (building it in-tree with nvcc if missing or stale)."""
    global _lib
    if _lib is not None:
        return _lib
    if build_if_missing:
        from . import _build
        try:
            _build.build()
        except Exception:
            if not os.path.exists(_SO):
                raise
    if not os.path.exists(_SO):
        raise ImportError("paper_2003_04776_b200: CUDA library %s is missing (run __graft_entry__.build())" % _SO)
    lib = ctypes.CDLL(_SO)
    vp, ci = ctypes.c_void_p, ctypes.c_int
    sig = {
        "zz_get_unique_id": ([vp], ci),
        "zz_init": ([ci, ci, ci, vp], ci),
        "zz_set_shard": ([ci, ci], ci),
        "zz_shard_columns": ([ci, vp, vp, ci, ci, vp], ci),
        "zz_set_stream": ([vp], ci),
        "zz_set_tile": ([ci], ci),
        "zz_set_timing": ([ci], ci),
        "zz_set_graphs": ([ci], ci),
        "zz_set_diag_team": ([ci], ci),
        "zz_set_fusion": ([ci], ci),
        "zz_set_lookahead": ([ci], ci),
        "zz_tgevc": ([ci, vp, ci, vp, ci, vp, vp, ci, vp], ci),
        "zz_tgevc_host": ([ci, vp, ci, vp, ci, vp, vp, ci, vp], ci),
        "zz_tgevc_back": ([ci, vp, ci, vp, ci, vp, vp, ci, vp, ci, vp], ci),
        "zz_tgevc_left": ([ci, vp, ci, vp, ci, vp, vp, ci, vp], ci),
        "zz_ztgevc": ([ci, vp, ci, vp, ci, vp, vp, ci, vp], ci),
        "zz_count_columns": ([ci, vp, ci, vp], ci),
        "zz_partition": ([ci, vp, ci, vp], ci),
        "zz_last_info": ([ctypes.POINTER(Info)], ci),
        "zz_finalize": ([], ci),
        "zz_status_string": ([ci], ctypes.c_char_p),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


def _check(st, what):
    if st != 0:
        raise ZZError(st, what)


_inited = {}


def init(device=None, nranks=1, rank=0, unique_id=None):
    """Create this thread's context on `device` (default: torch's current device) as rank
    `rank` of `nranks` (include/zz.h zz_init).  unique_id: the 128 bytes of get_unique_id()
    on rank 0 (required for nranks > 1; with nranks == 1 it creates a one-rank communicator)."""
    import torch
    if device is None:
        device = torch.cuda.current_device()
    lib = load()
    uid = None
    if unique_id is not None:
        if len(unique_id) != 128:
            raise ValueError("unique_id must be 128 bytes")
        uid = ctypes.create_string_buffer(bytes(unique_id), 128)
    _check(lib.zz_init(int(device), int(nranks), int(rank), uid), "zz_init")
    _inited[device] = True
    return device


def get_unique_id():
    """128-byte NCCL unique id (rank 0; ship it to the other ranks)."""
    buf = ctypes.create_string_buffer(128)
    _check(load().zz_get_unique_id(buf), "zz_get_unique_id")
    return buf.raw


def init_distributed(rank, world, device=None, group=None):
    """Multi-GPU context: rank 0 creates the NCCL id, torch.distributed ships it (plumbing
    only), every rank calls zz_init(device, world, rank, id).  Collective."""
    import torch.distributed as dist
    obj = [get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return init(device, world, rank, obj[0])


def set_shard(p, P):
    """One-GPU emulation of rank p's share of P (include/zz.h zz_set_shard); (0, 1) resets."""
    _check(load().zz_set_shard(int(p), int(P)), "zz_set_shard")


def shard_columns(sub, m, P, p, select=None):
    """Global output columns owned by shard p of P (host-only ownership rule of the library,
    include/zz.h zz_shard_columns)."""
    import numpy as np
    s = np.ascontiguousarray(np.asarray(sub, dtype=np.float64).reshape(-1))
    sel = _sel_array(select, m)
    out = np.zeros(max(m, 1), np.int32)
    n = load().zz_shard_columns(m, s.ctypes.data if s.size else None, None if sel is None else sel.ctypes.data,
                                int(P), int(p), out.ctypes.data)
    if n < 0:
        raise ZZError(n, "zz_shard_columns")
    return out[:n].copy()


def set_tile(mb):
    _check(load().zz_set_tile(int(mb)), "zz_set_tile")


def set_fusion(k):
    """Step grouping of the wavefront: 1 .. 6 consecutive steps per update (default 4)."""
    _check(load().zz_set_fusion(int(k)), "zz_set_fusion")


def set_lookahead(mode):
    """Lookahead schedule: 0 off, 1 automatic (default), 2 on (include/zz.h)."""
    _check(load().zz_set_lookahead(int(mode)), "zz_set_lookahead")


def set_graphs(on):
    """CUDA-graph capture and replay of the wavefront (include/zz.h zz_set_graphs)."""
    _check(load().zz_set_graphs(1 if on else 0), "zz_set_graphs")


def set_diag_team(w=0):
    """Warps per diagonal-solve task (include/zz.h zz_set_diag_team; 0 = automatic).
    Results are bitwise independent of it."""
    _check(load().zz_set_diag_team(int(w)), "zz_set_diag_team")


def set_timing(on):
    _check(load().zz_set_timing(1 if on else 0), "zz_set_timing")


def last_info():
    inf = Info()
    _check(load().zz_last_info(ctypes.byref(inf)), "zz_last_info")
    return inf.as_dict()


def last_views():
    """Host copies of the device views of the last call (include/zz.h zz_info_t): a dict of
    numpy arrays logmax (L_c), a, b, beta, n_sel entries each, or None where the view is NULL."""
    import numpy as np
    inf = Info()
    _check(load().zz_last_info(ctypes.byref(inf)), "zz_last_info")
    n = inf.n_sel
    out = {}
    for k in ("logmax", "a", "b", "beta"):
        ptr = getattr(inf, "d_" + k)
        out[k] = None if not ptr else np.frombuffer(_d2h(ptr, 8 * n), dtype=np.float64).copy()
    return out


def _ld_colmajor(A, m, what):
    """leading dimension of a column-major 2-D tensor/array (stride(0) == 1)"""
    if A.dim() != 2 if hasattr(A, "dim") else A.ndim != 2:
        raise ValueError("%s must be 2-D" % what)
    st = A.stride() if hasattr(A, "stride") and callable(A.stride) else tuple(s // 8 for s in A.strides)
    if A.shape[0] != m:
        raise ValueError("%s must have %d rows" % (what, m))
    if A.shape[1] > 1 and st[0] != 1:
        raise ValueError("%s must be column-major (stride(0) == 1); use colmajor()" % what)
    return max(st[1] if A.shape[1] > 1 else m, 1)


def colmajor(A):
    """Column-major copy/view of a 2-D torch tensor (element (i,j) at i + j*ld)."""
    return A.t().contiguous().t()


def empty_colmajor(m, n, device="cuda", dtype=None, pin_memory=False):
    import torch
    dtype = dtype or torch.float64
    if device == "cpu":
        return torch.empty((n, m), dtype=dtype, pin_memory=pin_memory).t()
    return torch.empty((n, m), dtype=dtype, device=device).t()


def _sel_array(select, m):
    if select is None:
        return None
    import numpy as np
    s = np.ascontiguousarray(np.asarray(select.cpu() if hasattr(select, "cpu") else select, dtype=np.int32))
    if s.size != m:
        raise ValueError("select must have m entries")
    return s


def count_columns(S_host, select=None):
    """Number of output columns for (S, select); S on the host (numpy, column-major)."""
    import numpy as np
    S_host = np.asfortranarray(S_host, dtype=np.float64)
    m = S_host.shape[0]
    sel = _sel_array(select, m)
    n = load().zz_count_columns(m, S_host.ctypes.data, max(m, 1), None if sel is None else sel.ctypes.data)
    if n < 0:
        raise ZZError(n, "zz_count_columns")
    return n


def partition(sub, m, mb):
    """Host tile partition (reading R12): returns tile_start[0..M]."""
    import numpy as np
    s = np.ascontiguousarray(np.asarray(sub, dtype=np.float64).reshape(-1))
    out = np.zeros(m // max(mb - 1, 1) + 3, dtype=np.int32)
    M = load().zz_partition(m, s.ctypes.data if s.size else None, mb, out.ctypes.data)
    if M < 0:
        raise ZZError(M, "zz_partition")
    return out[:M + 1].copy()


def tgevc(S, T, select=None, X=None, col_scale_exp=None, stream=None, n_sel=None):
    """Selected right eigenvectors of the Schur pencil (S, T) on the GPU.

    S, T: CUDA float64 tensors, m x m, column-major (stride(0) == 1); never written.
    select: host int array of length m or None.  Returns (X, col_scale_exp): X is an
    m x n_sel column-major CUDA tensor, col_scale_exp int32 (implementation-defined
    exponents, include/zz.h)."""
    import torch
    lib = load()
    m = S.shape[0]
    if not (S.is_cuda and T.is_cuda):
        raise ValueError("S and T must be CUDA tensors (no CPU fallback)")
    if S.dtype != torch.float64 or T.dtype != torch.float64:
        raise ValueError("S and T must be float64")
    dev = S.device.index
    if dev not in _inited:
        init(dev)
    lds = _ld_colmajor(S, m, "S")
    ldt = _ld_colmajor(T, m, "T")
    sel = _sel_array(select, m)
    if n_sel is None:
        if sel is None:
            n_sel = m
        else:
            # count on the host from the subdiagonal
            sub = torch.diagonal(S, -1).cpu().numpy() if m > 1 else []
            n_sel = _count_from_sub(sub, m, sel)
    if X is None:
        X = empty_colmajor(m, max(n_sel, 1), device=S.device)[:, :n_sel]
    ldx = _ld_colmajor(X, m, "X") if n_sel > 0 else max(m, 1)
    if col_scale_exp is None:
        col_scale_exp = torch.empty(max(n_sel, 1), dtype=torch.int32, device=S.device)[:n_sel]
    st = stream if stream is not None else torch.cuda.current_stream(S.device)
    _check(lib.zz_set_stream(ctypes.c_void_p(st.cuda_stream)), "zz_set_stream")
    r = lib.zz_tgevc(m, S.data_ptr(), lds, T.data_ptr(), ldt, None if sel is None else sel.ctypes.data,
                     X.data_ptr() if n_sel > 0 else ctypes.c_void_p(1), ldx,
                     col_scale_exp.data_ptr() if n_sel > 0 else None)
    _check(r, "zz_tgevc")
    return X, col_scale_exp


def tgevc_collective(m, S=None, T=None, select=None, X=None, col_scale_exp=None, stream=None):
    """zz_tgevc on a multi-rank context (init_distributed): rank 0 passes S, T (CUDA float64
    column-major) and gets (X, col_scale_exp); the other ranks pass only m (and the same
    select) and get (None, None)."""
    import torch
    lib = load()
    if S is not None:
        return tgevc(S, T, select=select, X=X, col_scale_exp=col_scale_exp, stream=stream)
    sel = _sel_array(select, m)
    st = stream if stream is not None else torch.cuda.current_stream()
    _check(lib.zz_set_stream(ctypes.c_void_p(st.cuda_stream)), "zz_set_stream")
    r = lib.zz_tgevc(int(m), None, 0, None, 0, None if sel is None else sel.ctypes.data, None, 0, None)
    _check(r, "zz_tgevc")
    return None, None


def tgevc_host_collective(m, S=None, T=None, select=None, X=None, col_scale_exp=None):
    """zz_tgevc_host on a multi-rank context: rank 0 passes host S, T (and X); others only m."""
    import torch
    lib = load()
    if S is not None:
        return tgevc_host(S, T, select=select, X=X, col_scale_exp=col_scale_exp)
    sel = _sel_array(select, m)
    _check(lib.zz_set_stream(ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)), "zz_set_stream")
    r = lib.zz_tgevc_host(int(m), None, 0, None, 0, None if sel is None else sel.ctypes.data, None, 0, None)
    _check(r, "zz_tgevc_host")
    return None, None


def ztgevc(S, T, select=None, X=None, col_scale_exp=None, stream=None):
    """Selected right eigenvectors of a COMPLEX Schur pencil (ZTGEVC analogue, include/zz.h
    zz_ztgevc): S, T complex128 CUDA tensors, m x m, column-major, Im T_jj = 0.  Returns
    (X, col_scale_exp), X an m x n_sel complex128 column-major CUDA tensor."""
    import torch
    lib = load()
    m = S.shape[0]
    if not (S.is_cuda and T.is_cuda):
        raise ValueError("S and T must be CUDA tensors (no CPU fallback)")
    if S.dtype != torch.complex128 or T.dtype != torch.complex128:
        raise ValueError("S and T must be complex128")
    dev = S.device.index
    if dev not in _inited:
        init(dev)
    lds = _ld_colmajor(S, m, "S")
    ldt = _ld_colmajor(T, m, "T")
    sel = _sel_array(select, m)
    n_sel = m if sel is None else int((sel != 0).sum())
    if X is None:
        X = torch.empty((max(n_sel, 1), m), dtype=torch.complex128, device=S.device).t()[:, :n_sel]
    ldx = _ld_colmajor(X, m, "X") if n_sel > 0 else max(m, 1)
    if col_scale_exp is None:
        col_scale_exp = torch.empty(max(n_sel, 1), dtype=torch.int32, device=S.device)[:n_sel]
    st = stream if stream is not None else torch.cuda.current_stream(S.device)
    _check(lib.zz_set_stream(ctypes.c_void_p(st.cuda_stream)), "zz_set_stream")
    r = lib.zz_ztgevc(m, S.data_ptr(), lds, T.data_ptr(), ldt, None if sel is None else sel.ctypes.data,
                      X.data_ptr() if n_sel > 0 else ctypes.c_void_p(1), ldx,
                      col_scale_exp.data_ptr() if n_sel > 0 else None)
    _check(r, "zz_ztgevc")
    return X, col_scale_exp


def tgevc_left(S, T, select=None, Y=None, col_scale_exp=None, stream=None, n_sel=None):
    """Selected LEFT eigenvectors y^H S = lambda y^H T (LAPACK xTGEVC SIDE='L'; include/zz.h
    zz_tgevc_left).  Arguments and result layout as tgevc()."""
    import torch
    lib = load()
    m = S.shape[0]
    if not (S.is_cuda and T.is_cuda):
        raise ValueError("S and T must be CUDA tensors (no CPU fallback)")
    if S.dtype != torch.float64 or T.dtype != torch.float64:
        raise ValueError("S and T must be float64")
    dev = S.device.index
    if dev not in _inited:
        init(dev)
    lds = _ld_colmajor(S, m, "S")
    ldt = _ld_colmajor(T, m, "T")
    sel = _sel_array(select, m)
    if n_sel is None:
        if sel is None:
            n_sel = m
        else:
            sub = torch.diagonal(S, -1).cpu().numpy() if m > 1 else []
            n_sel = _count_from_sub(sub, m, sel)
    if Y is None:
        Y = empty_colmajor(m, max(n_sel, 1), device=S.device)[:, :n_sel]
    ldy = _ld_colmajor(Y, m, "Y") if n_sel > 0 else max(m, 1)
    if col_scale_exp is None:
        col_scale_exp = torch.empty(max(n_sel, 1), dtype=torch.int32, device=S.device)[:n_sel]
    st = stream if stream is not None else torch.cuda.current_stream(S.device)
    _check(lib.zz_set_stream(ctypes.c_void_p(st.cuda_stream)), "zz_set_stream")
    r = lib.zz_tgevc_left(m, S.data_ptr(), lds, T.data_ptr(), ldt, None if sel is None else sel.ctypes.data,
                          Y.data_ptr() if n_sel > 0 else ctypes.c_void_p(1), ldy,
                          col_scale_exp.data_ptr() if n_sel > 0 else None)
    _check(r, "zz_tgevc_left")
    return Y, col_scale_exp


def tgevc_back(S, T, V, select=None, W=None, col_scale_exp=None, stream=None, n_sel=None):
    """Back-transformed eigenvectors W = V X (xTGEVC HOWMNY='B'; include/zz.h zz_tgevc_back).

    S, T, V: CUDA float64 column-major m x m tensors (V: the right Schur vectors of the QZ
    step, A = U S V^T, B = U T V^T); never written.  Returns (W, col_scale_exp), W m x n_sel
    column-major, each column (pair) normalised to max |w| = 1 (max |Re| + |Im| = 1)."""
    import torch
    lib = load()
    m = S.shape[0]
    if not (S.is_cuda and T.is_cuda and V.is_cuda):
        raise ValueError("S, T and V must be CUDA tensors (no CPU fallback)")
    if S.dtype != torch.float64 or T.dtype != torch.float64 or V.dtype != torch.float64:
        raise ValueError("S, T and V must be float64")
    dev = S.device.index
    if dev not in _inited:
        init(dev)
    lds = _ld_colmajor(S, m, "S")
    ldt = _ld_colmajor(T, m, "T")
    ldv = _ld_colmajor(V, m, "V")
    sel = _sel_array(select, m)
    if n_sel is None:
        if sel is None:
            n_sel = m
        else:
            sub = torch.diagonal(S, -1).cpu().numpy() if m > 1 else []
            n_sel = _count_from_sub(sub, m, sel)
    if W is None:
        W = empty_colmajor(m, max(n_sel, 1), device=S.device)[:, :n_sel]
    ldw = _ld_colmajor(W, m, "W") if n_sel > 0 else max(m, 1)
    if col_scale_exp is None:
        col_scale_exp = torch.empty(max(n_sel, 1), dtype=torch.int32, device=S.device)[:n_sel]
    st = stream if stream is not None else torch.cuda.current_stream(S.device)
    _check(lib.zz_set_stream(ctypes.c_void_p(st.cuda_stream)), "zz_set_stream")
    r = lib.zz_tgevc_back(m, S.data_ptr(), lds, T.data_ptr(), ldt, None if sel is None else sel.ctypes.data,
                          V.data_ptr(), ldv, W.data_ptr() if n_sel > 0 else ctypes.c_void_p(1), ldw,
                          col_scale_exp.data_ptr() if n_sel > 0 else None)
    _check(r, "zz_tgevc_back")
    return W, col_scale_exp


def _count_from_sub(sub, m, sel):
    n, j = 0, 0
    while j < m:
        two = j + 1 < m and sub[j] != 0.0
        sz = 2 if two else 1
        if sel is None or sel[j] or (two and sel[j + 1]):
            n += sz
        j += sz
    return n


def tgevc_host(S, T, select=None, X=None, col_scale_exp=None, device=None):
    """End-to-end variant: HOST S, T (column-major numpy arrays or CPU tensors, pinned memory
    recommended); returns host X (m x n_sel) and col_scale_exp.  Staging copies are part of
    the call (zz_tgevc_host)."""
    import numpy as np
    lib = load()
    if device is None:
        import torch
        device = torch.cuda.current_device()
    if device not in _inited:
        init(device)
    m = S.shape[0]

    def ptr_ld(A, what):
        if hasattr(A, "data_ptr"):
            return A.data_ptr(), _ld_colmajor(A, m, what)
        A = np.asarray(A)
        if A.dtype != np.float64 or A.ndim != 2 or A.shape[0] != m:
            raise ValueError("%s must be a float64 array with %d rows" % (what, m))
        if A.shape[1] <= 1 or A.flags.f_contiguous:
            return A.ctypes.data, max(m, 1)
        if A.strides[0] != 8 or A.strides[1] % 8:
            raise ValueError("%s must be column-major (element (i,j) at i + j*ld)" % what)
        return A.ctypes.data, A.strides[1] // 8

    sel = _sel_array(select, m)
    ps, lds = ptr_ld(S, "S")
    pt, ldt = ptr_ld(T, "T")
    if X is None:
        if hasattr(S, "data_ptr"):
            sub = np.diagonal(S.numpy(), -1) if m > 1 else []
        else:
            sub = np.diagonal(S, -1) if m > 1 else []
        n = _count_from_sub(sub, m, sel)
        X = np.zeros((m, max(n, 1)), order="F")[:, :n]
    n = X.shape[1]
    px, ldx = ptr_ld(X, "X") if n > 0 else (X.ctypes.data if hasattr(X, "ctypes") else X.data_ptr(), max(m, 1))
    if col_scale_exp is None:
        col_scale_exp = np.zeros(max(n, 1), np.int32)[:n]
    pe = col_scale_exp.ctypes.data if hasattr(col_scale_exp, "ctypes") else col_scale_exp.data_ptr()
    import torch
    _check(lib.zz_set_stream(ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)), "zz_set_stream")
    r = lib.zz_tgevc_host(m, ps, lds, pt, ldt, None if sel is None else sel.ctypes.data, px, ldx,
                          pe if n > 0 else None)
    _check(r, "zz_tgevc_host")
    return X, col_scale_exp


def finalize():
    if _lib is not None:
        _lib.zz_finalize()
    _inited.clear()
