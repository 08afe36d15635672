"""Thin ctypes binding of libbbf.so (include/bbf.h) — argument marshalling only.

Every step of the counting path runs in the library's CUDA kernels; this module converts
numpy arrays / torch CUDA tensors to pointers and status codes to exceptions.  There is no
CPU fallback: if libbbf.so is missing or no sm_100 device is present, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# BBF_LIB: load a diagnostic variant built by `python -m paper_2308_07932_b200.build --variant`
LIB_PATH = os.environ.get("BBF_LIB") or os.path.join(_HERE, "libbbf.so")

BBF_OK, BBF_EINVAL, BBF_ERANGE, BBF_EDUP, BBF_ENOMEM, BBF_ECUDA, BBF_ENCCL, BBF_EOVERFLOW = range(8)
STATUS_NAMES = {0: "BBF_OK", 1: "BBF_EINVAL", 2: "BBF_ERANGE", 3: "BBF_EDUP", 4: "BBF_ENOMEM",
                5: "BBF_ECUDA", 6: "BBF_ENCCL", 7: "BBF_EOVERFLOW"}
BBF_SIDE_U, BBF_SIDE_V = 0, 1
BBF_PTR_DEVICE = 1 << 0
BBF_POSITIVE_ONLY = 1 << 1
BBF_METRIC_BALANCED, BBF_METRIC_DEGREE = 0, 1
BBF_FORCE_SPARSE = 1 << 2
BBF_FORCE_DENSE = 1 << 3
BBF_OUTPUT_ASYNC = 1 << 4


class BBFError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS_NAMES.get(status, str(status))


class bbf_counts(C.Structure):
    _fields_ = [("balanced", C.c_uint64), ("unbalanced", C.c_uint64), ("total", C.c_uint64),
                ("wedges_G", C.c_uint64), ("ms_count", C.c_float)]


class bbf_pair(C.Structure):
    _fields_ = [("a", C.c_uint32), ("b", C.c_uint32), ("balanced", C.c_uint64),
                ("unbalanced", C.c_uint64)]


_lib = None


def lib():
    """Load libbbf.so (raises ImportError if it was not built — no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run python -m paper_2308_07932_b200.build")
        L = C.CDLL(LIB_PATH)
        P, u32, u64, i32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int
        L.bbf_abi_version.restype = i32
        L.bbf_last_error.restype = C.c_char_p
        L.bbf_nccl_unique_id.argtypes = [P]
        L.bbf_comm_init.argtypes = [P, i32, i32, i32, P]
        L.bbf_comm_free.argtypes = [P]
        L.bbf_graph_load_csr.argtypes = [u32, u32, P, P, P, u32, i32, P, P, P]
        L.bbf_graph_free.argtypes = [P]
        L.bbf_count_global.argtypes = [P, P]
        L.bbf_count_global_base.argtypes = [P, P]
        L.bbf_count_per_vertex.argtypes = [P, P, P, P, P, u32, P]
        L.bbf_count_pairs_topk.argtypes = [P, i32, u32, P, P, u32]
        L.bbf_graph_stats.argtypes = [P, P, P, P, P]
        L.bbf_graph_hybrid_core.argtypes = [P, P, P]
        L.bbf_count_per_edge.argtypes = [P, P, P, P, P, u32, P]
        L.bbf_topk_vertices.argtypes = [P, i32, i32, u32, P, P, P]
        L.bbf_estimate_global.argtypes = [u32, u32, P, P, P, u32, C.c_double, u32, u64, i32, P, P,
                                          P, P, P]
        L.bbf_upload_csr.argtypes = [u32, u32, P, P, P, i32, P]
        L.bbf_graph_load_upload.argtypes = [P, u32, P, P, P]
        L.bbf_upload_free.argtypes = [P]
        L.bbf_device_sync.argtypes = [i32]
        for f in ("bbf_nccl_unique_id", "bbf_comm_init", "bbf_comm_free", "bbf_graph_load_csr",
                  "bbf_graph_free", "bbf_count_global", "bbf_count_global_base", "bbf_count_per_vertex",
                  "bbf_count_pairs_topk", "bbf_graph_stats", "bbf_graph_hybrid_core", "bbf_count_per_edge", "bbf_estimate_global", "bbf_topk_vertices",
                  "bbf_upload_csr", "bbf_graph_load_upload", "bbf_upload_free", "bbf_device_sync"):
            getattr(L, f).restype = i32
        _lib = L
    return _lib


def _check(st: int):
    if st != BBF_OK:
        raise BBFError(st, lib().bbf_last_error().decode(errors="replace"))


def abi_version() -> int:
    return lib().bbf_abi_version()


def last_error() -> str:
    return lib().bbf_last_error().decode(errors="replace")


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(lib().bbf_nccl_unique_id(buf))
    return bytes(buf)


class Comm:
    def __init__(self, uid: bytes, nranks: int, rank: int, device: int):
        self.h = C.c_void_p()
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        _check(lib().bbf_comm_init(buf, nranks, rank, device, C.byref(self.h)))
        self.nranks, self.rank, self.device = nranks, rank, device

    def free(self):
        if self.h:
            lib().bbf_comm_free(self.h)
            self.h = C.c_void_p()


def _is_torch(x):
    return type(x).__module__.startswith("torch")


def _ptr(x):
    if x is None:
        return None
    if _is_torch(x):
        return C.c_void_p(x.data_ptr())
    return x.ctypes.data_as(C.c_void_p)


def device_sync(device: int = 0):
    """bbf_device_sync: completes BBF_OUTPUT_ASYNC copies (and all library work) on `device`."""
    _check(lib().bbf_device_sync(device))


class Upload:
    """bbf_upload_csr: an asynchronous host->device copy of a CSR (host numpy arrays or host torch
    tensors, pinned for a truly asynchronous copy); consumed by Graph.from_upload.  The host arrays
    are kept referenced until then."""

    def __init__(self, n_u, n_v, row_ptr, col, sign, device: int = 0):
        if _is_torch(row_ptr):
            assert not row_ptr.is_cuda and all(t.is_contiguous() for t in (row_ptr, col, sign))
            keep = (row_ptr, col, sign)
        else:
            keep = (np.ascontiguousarray(row_ptr, dtype=np.uint64),
                    np.ascontiguousarray(col, dtype=np.uint32),
                    np.ascontiguousarray(sign, dtype=np.uint8))
        self._keep = keep
        self.n_u, self.n_v, self.device = int(n_u), int(n_v), device
        self.h = C.c_void_p()
        _check(lib().bbf_upload_csr(self.n_u, self.n_v, _ptr(keep[0]), _ptr(keep[1]), _ptr(keep[2]),
                                    device, C.byref(self.h)))

    def free(self):
        if self.h:
            lib().bbf_upload_free(self.h)
            self.h = C.c_void_p()
        self._keep = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Graph:
    """A signed bipartite graph resident on one GPU (bbf_graph_load_csr).

    row_ptr (uint64, n_u+1), col (uint32), sign (uint8, 1 = positive): numpy arrays (host) or
    torch CUDA tensors (then BBF_PTR_DEVICE is passed)."""

    def __init__(self, n_u, n_v, row_ptr, col, sign, device: int = 0, stream=None,
                 comm: Comm | None = None, flags: int = 0):
        dev = _is_torch(row_ptr) and row_ptr.is_cuda
        if dev:
            flags |= BBF_PTR_DEVICE
            keep = (row_ptr, col, sign)
        elif _is_torch(row_ptr):  # host torch tensors (e.g. pinned): passed as they are
            assert all(t.is_contiguous() for t in (row_ptr, col, sign))
            keep = (row_ptr, col, sign)
        else:
            keep = (np.ascontiguousarray(row_ptr, dtype=np.uint64),
                    np.ascontiguousarray(col, dtype=np.uint32),
                    np.ascontiguousarray(sign, dtype=np.uint8))
        self._keep = keep
        self.h = C.c_void_p()
        self.n_u, self.n_v = int(n_u), int(n_v)
        st = C.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else (stream or 0))
        _check(lib().bbf_graph_load_csr(self.n_u, self.n_v, _ptr(keep[0]), _ptr(keep[1]),
                                        _ptr(keep[2]), flags, device, st,
                                        comm.h if comm else None, C.byref(self.h)))
        self._keep = None

    @classmethod
    def from_synth(cls, g, **kw):
        return cls(g.n_u, g.n_v, g.row_ptr, g.col, g.sign, **kw)

    @classmethod
    def from_upload(cls, up: Upload, stream=None, comm: Comm | None = None, flags: int = 0):
        """bbf_graph_load_upload: build from an Upload (consumed)."""
        self = cls.__new__(cls)
        self.h = C.c_void_p()
        self.n_u, self.n_v = up.n_u, up.n_v
        st = C.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else (stream or 0))
        hu, up.h = up.h, C.c_void_p()  # consumed by the call, whatever its status
        try:
            _check(lib().bbf_graph_load_upload(hu, flags, st, comm.h if comm else None, C.byref(self.h)))
        finally:
            up._keep = None
        return self

    def free(self):
        if self.h:
            lib().bbf_graph_free(self.h)
            self.h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.free()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def count_global(self) -> dict:
        c = bbf_counts()
        _check(lib().bbf_count_global(self.h, C.byref(c)))
        return dict(balanced=c.balanced, unbalanced=c.unbalanced, total=c.total,
                    wedges_G=c.wedges_G, ms_count=c.ms_count)

    def count_global_base(self) -> dict:
        """Global counts by Alg. 1 BB-Base (explicit pair checks; the paper's baseline)."""
        c = bbf_counts()
        _check(lib().bbf_count_global_base(self.h, C.byref(c)))
        return dict(balanced=c.balanced, unbalanced=c.unbalanced, total=c.total,
                    wedges_G=c.wedges_G, ms_count=c.ms_count)

    def count_per_vertex(self, out=None, flags: int = 0):
        """Returns (totals dict, bal_u, unb_u, bal_v, unb_v).  `out` may be a tuple of four
        int64/uint64 torch tensors: CUDA tensors (device outputs, BBF_PTR_DEVICE) or host
        tensors (e.g. pinned memory, written by the library's D2H copies)."""
        c = bbf_counts()
        if out is not None:
            bu, nu, bv, nv = out
            if bu.is_cuda:
                flags |= BBF_PTR_DEVICE
        else:
            bu, nu = np.zeros(self.n_u, np.uint64), np.zeros(self.n_u, np.uint64)
            bv, nv = np.zeros(self.n_v, np.uint64), np.zeros(self.n_v, np.uint64)
        _check(lib().bbf_count_per_vertex(self.h, _ptr(bu), _ptr(nu), _ptr(bv), _ptr(nv), flags,
                                          C.byref(c)))
        tot = dict(balanced=c.balanced, unbalanced=c.unbalanced, total=c.total,
                   wedges_G=c.wedges_G, ms_count=c.ms_count)
        return tot, bu, nu, bv, nv

    def count_per_edge(self, row_ptr, col, out=None):
        """Per-edge (totals, bal, unb) in the order of the CSR (row_ptr, col) — the graph's own
        edges, e.g. the arrays it was loaded from (numpy host arrays or CUDA tensors; `out` may be
        two CUDA tensors of nnz int64 for device outputs)."""
        c = bbf_counts()
        flags = 0
        if _is_torch(row_ptr) and row_ptr.is_cuda:
            flags |= BBF_PTR_DEVICE
            rp, cl = row_ptr, col
            bal, unb = out if out is not None else (None, None)
            assert bal is not None, "device CSR: pass out=(bal, unb) CUDA tensors"
        else:
            rp = np.ascontiguousarray(row_ptr, dtype=np.uint64)
            cl = np.ascontiguousarray(col, dtype=np.uint32)
            nnz = int(rp[-1]) if rp.size else 0
            bal, unb = np.zeros(nnz, np.uint64), np.zeros(nnz, np.uint64)
        _check(lib().bbf_count_per_edge(self.h, _ptr(rp), _ptr(cl), _ptr(bal), _ptr(unb), flags, C.byref(c)))
        tot = dict(balanced=c.balanced, unbalanced=c.unbalanced, total=c.total, wedges_G=c.wedges_G,
                   ms_count=c.ms_count)
        return tot, bal, unb

    def count_pairs_topk(self, k: int, side: int = BBF_SIDE_U, flags: int = 0):
        buf = (bbf_pair * max(int(k), 1))()
        n = C.c_uint32()
        _check(lib().bbf_count_pairs_topk(self.h, side, int(k), buf, C.byref(n), flags))
        return [(buf[i].a, buf[i].b, buf[i].balanced, buf[i].unbalanced) for i in range(n.value)]

    def topk_vertices(self, k: int, side: int = BBF_SIDE_U, metric: int = BBF_METRIC_BALANCED):
        """[(input id, score)] of the top-k vertices of `side` (bbf_topk_vertices)."""
        ids = np.zeros(max(int(k), 1), np.uint32)
        sc = np.zeros(max(int(k), 1), np.uint64)
        n = C.c_uint32()
        _check(lib().bbf_topk_vertices(self.h, side, metric, int(k), _ptr(ids), _ptr(sc), C.byref(n)))
        return [(int(ids[i]), int(sc[i])) for i in range(n.value)]

    def stats(self) -> dict:
        L, B = C.c_uint64(), C.c_uint64()
        ops = C.c_double()
        ms = C.c_float()
        _check(lib().bbf_graph_stats(self.h, C.byref(L), C.byref(B), C.byref(ops), C.byref(ms)))
        return dict(kernel_launches=L.value, algo_bytes=B.value, algo_ops=ops.value,
                    ms_main_kernel=ms.value)

    def hybrid_core(self) -> tuple:
        """(core_u, core_v) of the last count's hybrid dispatch, (0, 0) = none (bbf_graph_hybrid_core)."""
        a, b = C.c_uint32(), C.c_uint32()
        _check(lib().bbf_graph_hybrid_core(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value


def estimate_global(n_u, n_v, row_ptr, col, sign, rho: float, trials: int, seed: int = 0,
                    device: int = 0, stream=None, comm: Comm | None = None, flags: int = 0) -> dict:
    """SBESPAR sparsification estimate (bbf_estimate_global).  Returns dict(sampled_B, sampled_N
    (uint64 arrays), estimates (float64 array), mean, stddev).  The per-trial estimates come from
    the library; mean and stddev are summary statistics of those returned values, computed here
    for the caller (harness statistics, not a step of the method)."""
    dev = _is_torch(row_ptr) and row_ptr.is_cuda
    if dev:
        flags |= BBF_PTR_DEVICE
        keep = (row_ptr, col, sign)
    elif _is_torch(row_ptr):
        keep = (row_ptr, col, sign)
    else:
        keep = (np.ascontiguousarray(row_ptr, dtype=np.uint64),
                np.ascontiguousarray(col, dtype=np.uint32),
                np.ascontiguousarray(sign, dtype=np.uint8))
    sb, sn = np.zeros(trials, np.uint64), np.zeros(trials, np.uint64)
    est = np.zeros(trials, np.float64)
    st = C.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else (stream or 0))
    _check(lib().bbf_estimate_global(int(n_u), int(n_v), _ptr(keep[0]), _ptr(keep[1]), _ptr(keep[2]),
                                     flags, float(rho), int(trials), int(seed) & (2**64 - 1), device,
                                     st, comm.h if comm else None, _ptr(sb), _ptr(sn), _ptr(est)))
    return dict(sampled_B=sb, sampled_N=sn, estimates=est, mean=float(est.mean()),
                stddev=float(est.std(ddof=1)) if trials > 1 else 0.0)


# ABI-named aliases (same names as include/bbf.h)
bbf_abi_version = abi_version
bbf_last_error = last_error
bbf_nccl_unique_id = nccl_unique_id
bbf_comm_init = Comm
bbf_graph_load_csr = Graph


def bbf_graph_free(g: Graph):
    g.free()


def bbf_comm_free(c: Comm):
    c.free()


def bbf_count_global_base(g: Graph):
    return g.count_global_base()


def bbf_count_global(g: Graph):
    return g.count_global()


def bbf_count_per_vertex(g: Graph, out=None, flags: int = 0):
    return g.count_per_vertex(out, flags)


def bbf_count_pairs_topk(g: Graph, side: int, k: int, flags: int = 0):
    return g.count_pairs_topk(k, side, flags)


def bbf_count_per_edge(g: Graph, row_ptr, col, out=None):
    return g.count_per_edge(row_ptr, col, out)


def bbf_graph_stats(g: Graph):
    return g.stats()


def bbf_graph_hybrid_core(g: Graph):
    return g.hybrid_core()


bbf_estimate_global = estimate_global


def bbf_topk_vertices(g: Graph, side: int, metric: int, k: int):
    return g.topk_vertices(k, side, metric)
