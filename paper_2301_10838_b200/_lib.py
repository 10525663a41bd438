"""Thin ctypes binding of libmt_b200.so (include/mt.h) -- argument marshalling only.

Every step of the hot path runs in the library's sm_100a kernels; this module
only passes device pointers (torch tensors' ``data_ptr()``), sizes and the
current CUDA stream.  There is no CPU fallback: if the shared library is
missing or a call fails, an exception is raised.

Functions carry the C names (``mt_create``, ``mt_compute``, ``mt_diagram``,
...); ``MergeTree`` is a convenience owner of a context + its workspace.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# MT_LIBRARY: load another build of the same ABI (A/B experiments, scripts/ab_build.py)
SO_PATH = os.environ.get("MT_LIBRARY") or os.path.join(_PKG, "libmt_b200.so")

MT_OK, MT_ERR_INVALID_ARG, MT_ERR_TOO_LARGE, MT_ERR_NONFINITE, MT_ERR_CUDA = 0, 1, 2, 3, 4
MT_ERR_NCCL, MT_ERR_STATE, MT_ERR_CAPACITY, MT_ERR_WORKSPACE = 5, 6, 7, 8
MT_FLAG_SPLIT_TREE = 1

PAIR_DTYPE = np.dtype([("birth_v", "<u4"), ("death_v", "<u4"), ("birth", "<f4"), ("death", "<f4")])
PAIR64_DTYPE = np.dtype([("birth_v", "<u8"), ("death_v", "<u8"), ("birth", "<f4"), ("death", "<f4")])
TRIPLET64_DTYPE = np.dtype([("s", "<u8"), ("v", "<u8")])
FOREST_RECORD_BYTES = 32  # mt_forest_record
MT_SLAB_WIDE_IDS = 1      # mt_create_slab / mt_create_dist option

# every symbol include/mt.h declares (checked by tests/test_abi_cpu.py)
EXPORTS = ["mt_workspace_bytes", "mt_create", "mt_compute", "mt_set_diagram_output", "mt_diagram",
           "mt_diagram_view", "mt_last_error", "mt_last_launch_count", "mt_set_profiling", "mt_kernel_times",
           "mt_status_string", "mt_destroy", "mt_abi_version", "mt_set_stats", "mt_stats", "mt_slab_workspace_bytes",
           "mt_create_slab", "mt_compute_local", "mt_forest_view", "mt_forest_scratch_bytes", "mt_compute_global",
           "mt_filter_diagram", "mt_graph_workspace_bytes", "mt_create_graph", "mt_compute_graph",
           "mt_get_unique_id", "mt_dist_slab_bounds", "mt_dist_workspace_bytes", "mt_create_dist",
           "mt_compute_join_split", "mt_host_staging_bytes", "mt_compute_host", "mt_triplets64", "mt_diagram64"]


class MTError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: {status_string(status)} (status {status})")


_lib = None


def load(build_if_missing: bool = False):
    """Load the in-tree libmt_b200.so (fails loudly if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(SO_PATH):
        if build_if_missing:
            from . import build
            build.build()
        else:
            raise ImportError(f"{SO_PATH} is missing: run `python -m paper_2301_10838_b200.build` "
                              "(there is no CPU fallback)")
    lib = ctypes.CDLL(SO_PATH)
    u32p = ctypes.POINTER(ctypes.c_uint32)
    u64p = ctypes.POINTER(ctypes.c_uint64)
    vp = ctypes.c_void_p
    sig = {
        "mt_workspace_bytes": (ctypes.c_size_t, [u32p, ctypes.c_int]),
        "mt_create": (ctypes.c_int, [ctypes.POINTER(vp), u32p, ctypes.c_int, ctypes.c_int, vp, ctypes.c_size_t]),
        "mt_compute": (ctypes.c_int, [vp, vp, vp, ctypes.c_uint32, vp]),
        "mt_compute_join_split": (ctypes.c_int, [vp, vp, vp, vp, vp, vp]),
        "mt_host_staging_bytes": (ctypes.c_size_t, [vp]),
        "mt_compute_host": (ctypes.c_int, [vp, ctypes.c_uint32, vp, vp, vp, ctypes.c_uint64, vp, ctypes.c_uint32, vp,
                                           ctypes.c_size_t, vp]),
        "mt_set_diagram_output": (ctypes.c_int, [vp, vp, ctypes.c_uint64]),
        "mt_diagram": (ctypes.c_int, [vp, vp, ctypes.c_uint64, u64p, u64p, vp]),
        "mt_diagram_view": (ctypes.c_int, [vp, ctypes.POINTER(vp), u64p, u64p, vp]),
        "mt_last_error": (ctypes.c_int, [vp, vp]),
        "mt_filter_diagram": (ctypes.c_int, [vp, ctypes.c_float, vp, ctypes.c_uint64, u64p, u64p, vp]),
        "mt_graph_workspace_bytes": (ctypes.c_size_t, [ctypes.c_uint32, ctypes.c_uint64]),
        "mt_create_graph": (ctypes.c_int, [ctypes.POINTER(vp), ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int, vp,
                                           ctypes.c_size_t]),
        "mt_compute_graph": (ctypes.c_int, [vp, vp, vp, vp, vp, ctypes.c_uint32, vp]),
        "mt_last_launch_count": (ctypes.c_uint32, [vp]),
        "mt_set_profiling": (ctypes.c_int, [vp, ctypes.c_int]),
        "mt_kernel_times": (ctypes.c_int, [vp, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(ctypes.c_float),
                                           ctypes.c_int]),
        "mt_status_string": (ctypes.c_char_p, [ctypes.c_int]),
        "mt_set_stats": (ctypes.c_int, [vp, ctypes.c_int]),
        "mt_stats": (ctypes.c_int, [vp, u64p, ctypes.c_int, vp]),
        "mt_destroy": (None, [vp]),
        "mt_slab_workspace_bytes": (ctypes.c_size_t, [u32p, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32]),
        "mt_create_slab": (ctypes.c_int, [ctypes.POINTER(vp), u32p, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32,
                                          ctypes.c_uint32, ctypes.c_int, vp, ctypes.c_size_t]),
        "mt_compute_local": (ctypes.c_int, [vp, vp, vp, ctypes.c_uint32, vp]),
        "mt_forest_view": (ctypes.c_int, [vp, ctypes.POINTER(vp), u64p, vp]),
        "mt_forest_scratch_bytes": (ctypes.c_size_t, [ctypes.c_uint64]),
        "mt_compute_global": (ctypes.c_int, [vp, vp, u64p, u32p, ctypes.c_uint32, vp, ctypes.c_size_t, vp, vp]),
        "mt_triplets64": (ctypes.c_int, [vp, vp, ctypes.c_uint64, ctypes.c_uint64, vp, vp]),
        "mt_diagram64": (ctypes.c_int, [vp, vp, ctypes.c_uint64, u64p, u64p, vp]),
        "mt_abi_version": (ctypes.c_int, []),
        "mt_get_unique_id": (ctypes.c_int, [ctypes.c_void_p]),
        "mt_dist_slab_bounds": (ctypes.c_int, [ctypes.c_uint32, ctypes.c_int, u32p]),
        "mt_dist_workspace_bytes": (ctypes.c_size_t, [u32p, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
        "mt_create_dist": (ctypes.c_int, [ctypes.POINTER(vp), u32p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_void_p, ctypes.c_uint32, ctypes.c_int, vp, ctypes.c_size_t]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def status_string(st: int) -> str:
    try:
        return load().mt_status_string(st).decode()
    except ImportError:
        return f"status {st}"


def _dims(dims):
    return (ctypes.c_uint32 * 3)(*[int(d) for d in dims])


def _stream_handle(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _check(st, where):
    if st != MT_OK:
        raise MTError(st, where)


# ---- C-named wrappers -------------------------------------------------------

def mt_workspace_bytes(dims, conn: int) -> int:
    return int(load().mt_workspace_bytes(_dims(dims), int(conn)))


def mt_create(dims, conn: int, device: int, workspace_ptr: int, workspace_bytes: int):
    h = ctypes.c_void_p()
    _check(load().mt_create(ctypes.byref(h), _dims(dims), int(conn), int(device), ctypes.c_void_p(workspace_ptr),
                            ctypes.c_size_t(workspace_bytes)), "mt_create")
    return h


def mt_compute(ctx, f_ptr: int, triplets_ptr: int, flags: int = 0, stream=None):
    _check(load().mt_compute(ctx, ctypes.c_void_p(f_ptr), ctypes.c_void_p(triplets_ptr), int(flags),
                             _stream_handle(stream)), "mt_compute")


def mt_compute_join_split(ctx_join, ctx_split, f_ptr: int, tj_ptr: int, ts_ptr: int, stream=None):
    _check(load().mt_compute_join_split(ctx_join, ctx_split, ctypes.c_void_p(f_ptr), ctypes.c_void_p(tj_ptr),
                                        ctypes.c_void_p(ts_ptr), _stream_handle(stream)), "mt_compute_join_split")


def mt_host_staging_bytes(ctx) -> int:
    return int(load().mt_host_staging_bytes(ctx))


def mt_compute_host(ctx, f_ptrs, T_ptrs, rec_ptrs, rec_cap: int, flags: int, staging_ptr: int, staging_bytes: int,
                    stream=None):
    """Host->host steps (pointers to pinned host buffers); returns [(n_pairs, n_essential)] per field."""
    k = len(f_ptrs)
    arr = lambda xs: (ctypes.c_void_p * max(k, 1))(*[ctypes.c_void_p(x) for x in xs])
    counts = (ctypes.c_uint64 * (2 * max(k, 1)))()
    _check(load().mt_compute_host(ctx, k, arr(f_ptrs), arr(T_ptrs), arr(rec_ptrs), ctypes.c_uint64(rec_cap), counts,
                                  int(flags), ctypes.c_void_p(staging_ptr), ctypes.c_size_t(staging_bytes),
                                  _stream_handle(stream)), "mt_compute_host")
    return [(int(counts[2 * i]), int(counts[2 * i + 1])) for i in range(k)]


def mt_set_diagram_output(ctx, buf_ptr: int, capacity: int):
    _check(load().mt_set_diagram_output(ctx, ctypes.c_void_p(buf_ptr), ctypes.c_uint64(capacity)),
           "mt_set_diagram_output")


def mt_diagram(ctx, out_ptr: int = 0, capacity: int = 0, stream=None):
    """Returns (status, n_pairs, n_essential); raises only on CUDA/state errors."""
    npairs, ness = ctypes.c_uint64(0), ctypes.c_uint64(0)
    st = load().mt_diagram(ctx, ctypes.c_void_p(out_ptr or None), ctypes.c_uint64(capacity), ctypes.byref(npairs),
                           ctypes.byref(ness), _stream_handle(stream))
    if st in (MT_ERR_CUDA, MT_ERR_STATE, MT_ERR_INVALID_ARG):
        raise MTError(st, "mt_diagram")
    return st, npairs.value, ness.value


def mt_diagram_view(ctx, stream=None):
    ptr, npairs, ness = ctypes.c_void_p(), ctypes.c_uint64(0), ctypes.c_uint64(0)
    st = load().mt_diagram_view(ctx, ctypes.byref(ptr), ctypes.byref(npairs), ctypes.byref(ness),
                                _stream_handle(stream))
    if st in (MT_ERR_CUDA, MT_ERR_STATE, MT_ERR_INVALID_ARG):
        raise MTError(st, "mt_diagram_view")
    return st, ptr.value, npairs.value, ness.value


def mt_filter_diagram(ctx, eps: float, out_ptr: int, capacity: int, stream=None):
    """Returns (status, n_pairs_kept, n_essential)."""
    a, b = ctypes.c_uint64(0), ctypes.c_uint64(0)
    st = load().mt_filter_diagram(ctx, ctypes.c_float(eps), ctypes.c_void_p(out_ptr or None),
                                  ctypes.c_uint64(capacity), ctypes.byref(a), ctypes.byref(b), _stream_handle(stream))
    if st in (MT_ERR_CUDA, MT_ERR_STATE, MT_ERR_INVALID_ARG):
        raise MTError(st, "mt_filter_diagram")
    return st, a.value, b.value


def mt_last_error(ctx, stream=None) -> int:
    return int(load().mt_last_error(ctx, _stream_handle(stream)))


def mt_last_launch_count(ctx) -> int:
    return int(load().mt_last_launch_count(ctx))


def mt_set_profiling(ctx, enable: bool):
    _check(load().mt_set_profiling(ctx, int(bool(enable))), "mt_set_profiling")


def mt_kernel_times(ctx, max_entries: int = 16):
    names = (ctypes.c_char_p * max_entries)()
    ms = (ctypes.c_float * max_entries)()
    k = load().mt_kernel_times(ctx, names, ms, max_entries)
    return [(names[i].decode(), float(ms[i])) for i in range(k)]


STAT_NAMES = ["edges", "skipped", "pre_hops", "merge_iters", "cas_fail", "repair_hops", "tile_edges",
              "tile_hops", "tile_iters", "tile_repair_hops", "tile_compress_hops", "cyc_load", "cyc_descent",
              "cyc_compress", "cyc_merge", "cyc_repair", "cyc_write", "cyc_list", "tile_pairs", "queued"]


def mt_set_stats(ctx, enable: bool):
    _check(load().mt_set_stats(ctx, int(bool(enable))), "mt_set_stats")


def mt_stats(ctx, stream=None):
    out = (ctypes.c_uint64 * 24)()
    k = load().mt_stats(ctx, out, 24, _stream_handle(stream))
    return {name: int(out[i]) for i, name in enumerate(STAT_NAMES) if i < k}


def mt_destroy(ctx):
    load().mt_destroy(ctx)


# ---- multi-GPU z-slab entry points (include/mt.h) ---------------------------

def mt_slab_workspace_bytes(dims, conn: int, z_begin: int, z_end: int) -> int:
    return int(load().mt_slab_workspace_bytes(_dims(dims), int(conn), int(z_begin), int(z_end)))


def mt_create_slab(dims, conn: int, z_begin: int, z_end: int, device: int, workspace_ptr: int, workspace_bytes: int,
                   options: int = 0):
    h = ctypes.c_void_p()
    _check(load().mt_create_slab(ctypes.byref(h), _dims(dims), int(conn), int(z_begin), int(z_end), int(options),
                                 int(device), ctypes.c_void_p(workspace_ptr), ctypes.c_size_t(workspace_bytes)),
           "mt_create_slab")
    return h


def mt_compute_local(ctx, f_ptr: int, triplets_ptr: int, flags: int = 0, stream=None):
    _check(load().mt_compute_local(ctx, ctypes.c_void_p(f_ptr), ctypes.c_void_p(triplets_ptr), int(flags),
                                   _stream_handle(stream)), "mt_compute_local")


def mt_forest_view(ctx, stream=None):
    ptr, n = ctypes.c_void_p(), ctypes.c_uint64(0)
    _check(load().mt_forest_view(ctx, ctypes.byref(ptr), ctypes.byref(n), _stream_handle(stream)), "mt_forest_view")
    return ptr.value, n.value


def mt_forest_scratch_bytes(n_all: int) -> int:
    return int(load().mt_forest_scratch_bytes(ctypes.c_uint64(n_all)))


def mt_compute_global(ctx, all_ptr: int, counts, z_bounds, scratch_ptr: int, scratch_bytes: int,
                      triplets_ptr: int, stream=None):
    """``counts``: records per slab (the gathered array holds them in slab order)."""
    if len(counts) != len(z_bounds) - 1:
        raise ValueError("one record count per slab")
    zb = (ctypes.c_uint32 * len(z_bounds))(*[int(z) for z in z_bounds])
    cn = (ctypes.c_uint64 * len(counts))(*[int(c) for c in counts])
    _check(load().mt_compute_global(ctx, ctypes.c_void_p(all_ptr or None), cn, zb,
                                    len(z_bounds) - 1, ctypes.c_void_p(scratch_ptr), ctypes.c_size_t(scratch_bytes),
                                    ctypes.c_void_p(triplets_ptr), _stream_handle(stream)), "mt_compute_global")


def mt_triplets64(ctx, triplets_ptr: int, first: int, count: int, out_ptr: int, stream=None):
    _check(load().mt_triplets64(ctx, ctypes.c_void_p(triplets_ptr or None), ctypes.c_uint64(first),
                                ctypes.c_uint64(count), ctypes.c_void_p(out_ptr or None), _stream_handle(stream)),
           "mt_triplets64")


def mt_diagram64(ctx, out_ptr: int, capacity: int, stream=None):
    """Syncs; (status, n_pairs, n_essential); records copied to out_ptr (device) when non-zero."""
    a, b = ctypes.c_uint64(0), ctypes.c_uint64(0)
    st = load().mt_diagram64(ctx, ctypes.c_void_p(out_ptr or None), ctypes.c_uint64(capacity), ctypes.byref(a),
                             ctypes.byref(b), _stream_handle(stream))
    return st, a.value, b.value


# ---- multi-GPU with the NCCL exchange inside the library -------------------------

def mt_get_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(load().mt_get_unique_id(buf), "mt_get_unique_id")
    return bytes(buf)


def mt_dist_slab_bounds(nz: int, nranks: int) -> list[int]:
    b = (ctypes.c_uint32 * (int(nranks) + 1))()
    _check(load().mt_dist_slab_bounds(int(nz), int(nranks), b), "mt_dist_slab_bounds")
    return [int(x) for x in b]


def mt_dist_workspace_bytes(dims, conn: int, rank: int, nranks: int) -> int:
    return int(load().mt_dist_workspace_bytes(_dims(dims), int(conn), int(rank), int(nranks)))


def mt_create_dist(dims, conn: int, rank: int, nranks: int, nccl_id: bytes, device: int, workspace_ptr: int,
                   workspace_bytes: int, options: int = 0):
    if len(nccl_id) != 128:
        raise ValueError("an NCCL unique id is 128 bytes")
    h = ctypes.c_void_p()
    idbuf = (ctypes.c_uint8 * 128)(*nccl_id)
    _check(load().mt_create_dist(ctypes.byref(h), _dims(dims), int(conn), int(rank), int(nranks), idbuf,
                                 int(options), int(device), ctypes.c_void_p(workspace_ptr),
                                 ctypes.c_size_t(workspace_bytes)),
           "mt_create_dist")
    return h


# ---- explicit graphs ------------------------------------------------------------

def mt_graph_workspace_bytes(n: int, n_adj: int) -> int:
    return int(load().mt_graph_workspace_bytes(int(n), ctypes.c_uint64(n_adj)))


def mt_create_graph(n: int, n_adj: int, device: int, workspace_ptr: int, workspace_bytes: int):
    h = ctypes.c_void_p()
    _check(load().mt_create_graph(ctypes.byref(h), int(n), ctypes.c_uint64(n_adj), int(device),
                                  ctypes.c_void_p(workspace_ptr), ctypes.c_size_t(workspace_bytes)), "mt_create_graph")
    return h


def mt_compute_graph(ctx, f_ptr: int, row_ptr: int, col_ptr: int, triplets_ptr: int, flags: int = 0, stream=None):
    _check(load().mt_compute_graph(ctx, ctypes.c_void_p(f_ptr), ctypes.c_void_p(row_ptr),
                                   ctypes.c_void_p(col_ptr or None), ctypes.c_void_p(triplets_ptr), int(flags),
                                   _stream_handle(stream)), "mt_compute_graph")


class GraphMergeTree:
    """A context for an explicit graph (CSR adjacency, both directions listed) on one device."""

    def __init__(self, n: int, n_adj: int, device=None):
        import torch
        self.n, self.n_adj = int(n), int(n_adj)
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else int(device)) \
            if not isinstance(device, torch.device) else device
        self.device = dev
        nbytes = mt_graph_workspace_bytes(self.n, self.n_adj)
        self.workspace = torch.empty(nbytes + 256, dtype=torch.uint8, device=dev)
        ptr = (self.workspace.data_ptr() + 255) // 256 * 256
        self.ctx = mt_create_graph(self.n, self.n_adj, dev.index, ptr, nbytes)

    def __del__(self):
        ctx = getattr(self, "ctx", None)
        if ctx is not None and _lib is not None:
            _lib.mt_destroy(ctx)
            self.ctx = None

    def compute(self, f, row, col, split: bool = False, triplets=None, stream=None):
        """f float32[n], row int64[n+1], col int32[row[n]] CUDA tensors -> int64 triplets (async)."""
        import torch
        if f.numel() != self.n or row.numel() != self.n + 1 or col.numel() > self.n_adj:
            raise ValueError("graph sizes do not match the context")
        for t, dts, name in ((f, (torch.float32,), "f"), (row, (torch.int64, torch.uint64), "row"),
                             (col, (torch.int32, torch.uint32), "col")):
            if t.dtype not in dts or not t.is_cuda or not t.is_contiguous() or t.device != self.device:
                raise ValueError(f"{name} must be a contiguous {dts[0]} tensor on {self.device}")
        if triplets is None:
            triplets = torch.empty(self.n, dtype=torch.int64, device=f.device)
        mt_compute_graph(self.ctx, f.data_ptr(), row.data_ptr(), col.data_ptr() if col.numel() else 0,
                         triplets.data_ptr(), MT_FLAG_SPLIT_TREE if split else 0, stream)
        return triplets

    diagram = None  # set below (shared with MergeTree)


# ---- convenience owner --------------------------------------------------------

class MergeTree:
    """A context for one grid shape on one device, owning its workspace (a torch tensor)."""

    def __init__(self, dims, conn: int = 6, device=None):
        import torch
        self.dims = tuple(int(d) for d in dims)
        self.conn = int(conn)
        self.n = self.dims[0] * self.dims[1] * self.dims[2]
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else int(device)) \
            if not isinstance(device, torch.device) else device
        self.device = dev
        nbytes = mt_workspace_bytes(self.dims, self.conn)
        if nbytes == 0:
            raise MTError(MT_ERR_INVALID_ARG, "mt_workspace_bytes")
        self.workspace = torch.empty(nbytes + 256, dtype=torch.uint8, device=dev)
        ptr = self.workspace.data_ptr()
        self._ws_ptr = (ptr + 255) // 256 * 256
        self.ctx = mt_create(self.dims, self.conn, dev.index, self._ws_ptr, nbytes)
        self._out = None

    def __del__(self):
        ctx = getattr(self, "ctx", None)
        if ctx is not None and _lib is not None:
            _lib.mt_destroy(ctx)
            self.ctx = None

    def set_diagram_output(self, buf):
        """Register a (k, 4) int32 CUDA tensor as the zero-copy diagram target (None detaches)."""
        self._out = buf
        mt_set_diagram_output(self.ctx, buf.data_ptr() if buf is not None else 0, buf.shape[0] if buf is not None else 0)

    def compute(self, f, triplets=None, split: bool = False, stream=None):
        """f: float32 CUDA tensor with n elements (x fastest).  Returns the int64 tensor
        holding the uint64 cells s << 32 | v (asynchronous)."""
        import torch
        if f.dtype != torch.float32 or not f.is_cuda or not f.is_contiguous() or f.numel() != self.n:
            raise ValueError("f must be a contiguous float32 CUDA tensor with nx*ny*nz elements")
        if triplets is None:
            triplets = torch.empty(self.n, dtype=torch.int64, device=f.device)
        mt_compute(self.ctx, f.data_ptr(), triplets.data_ptr(), MT_FLAG_SPLIT_TREE if split else 0, stream)
        return triplets

    def diagram(self, stream=None, copy: bool = True):
        """Synchronises; returns (records (k,4) int32 CUDA tensor, n_pairs, n_essential)."""
        import torch
        st, ptr, npairs, ness = mt_diagram_view(self.ctx, stream)
        if st != MT_OK:
            raise MTError(st, "mt_diagram")
        k = npairs + ness
        out = torch.empty((k, 4), dtype=torch.int32, device=self.device)
        if k:
            st, a, b = mt_diagram(self.ctx, out.data_ptr(), k, stream)
            _check(st, "mt_diagram")
        return out, npairs, ness

    def filter_diagram(self, eps: float, stream=None):
        """Pairs with persistence > eps (+ essential classes): ((k,4) int32 CUDA tensor, n_pairs, n_ess)."""
        import torch
        st, ptr, npairs, ness = mt_diagram_view(self.ctx, stream)
        cap = max(1, npairs + ness)
        out = torch.empty((cap, 4), dtype=torch.int32, device=self.device)
        st, a, b = mt_filter_diagram(self.ctx, eps, out.data_ptr(), cap, stream)
        _check(st, "mt_filter_diagram")
        return out[: a + b], a, b

    def last_launch_count(self):
        return mt_last_launch_count(self.ctx)


def join_split(mt_join: "MergeTree", mt_split: "MergeTree", f, stream=None):
    """Merge and split tree of f from one read of f (mt_compute_join_split): returns the two
    int64 triplet tensors; each context's diagram() then reports its tree's diagram."""
    import torch
    if f.dtype != torch.float32 or not f.is_cuda or not f.is_contiguous() or f.numel() != mt_join.n:
        raise ValueError("f must be a contiguous float32 CUDA tensor with nx*ny*nz elements")
    tj = torch.empty(mt_join.n, dtype=torch.int64, device=f.device)
    ts = torch.empty(mt_split.n, dtype=torch.int64, device=f.device)
    mt_compute_join_split(mt_join.ctx, mt_split.ctx, f.data_ptr(), tj.data_ptr(), ts.data_ptr(), stream)
    return tj, ts


GraphMergeTree.diagram = MergeTree.diagram
GraphMergeTree.filter_diagram = MergeTree.filter_diagram


def pairs_to_numpy(records) -> np.ndarray:
    """(k, 4) int32 tensor -> structured numpy array with PAIR_DTYPE."""
    a = records.detach().cpu().contiguous().numpy()
    return a.view(PAIR_DTYPE).reshape(-1)
