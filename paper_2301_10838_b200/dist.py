"""Multi-GPU z-slab decomposition: one process per GPU.

Rank r owns planes [z_bounds[r], z_bounds[r+1]) of the global grid (3D, 6-connectivity).
Two transports for the one exchange step:
  * ``transport="nccl"`` (the product path): ``mt_create_dist`` -- the library owns an NCCL
    communicator and ``mt_compute`` runs local phase -> NCCL exchange -> global phase itself;
    Python only broadcasts rank 0's 128-byte NCCL unique id.
  * ``transport="torch"`` (pluggable, for gloo and tests): the three-call ABI
      1. ``mt_compute_local``   -- the slab's merge tree + its boundary forest (device kernels);
      2. all-gather of the forest records over the process group (``torch.distributed``);
      3. ``mt_compute_global``  -- every rank merges all inter-slab edges on the gathered
         forest, writes back its cells, repairs its slab and extracts its part of the diagram.
The triplets hold global ids (32-bit mode) or the context's view ids (wide mode, SURVEY.md 8f row
f3: global grids past 2^32 vertices, or ``wide=True``), which ``triplets64`` / ``diagram64``
translate to 64-bit global ids; the finite pairs of rank r are the branches born in its slab
(ascending), so concatenating the ranks in order gives the single-GPU diagram.
This module is plumbing (argument marshalling + the collective); all computation runs in
libmt_b200.so.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib

RECORD_BYTES = _lib.FOREST_RECORD_BYTES


def slab_bounds(nz: int, nranks: int) -> list[int]:
    """z boundaries of ``nranks`` slabs covering ``nz`` planes (the library's rule,
    ``mt_dist_slab_bounds``: as equal as possible, on multiples of the tile depth 8 when
    nz >= 8 nranks)."""
    if nranks < 1 or nranks > nz or nranks > 64:
        raise ValueError("need 1 <= nranks <= min(nz, 64)")
    return _lib.mt_dist_slab_bounds(nz, nranks)


def allgather_varsize(t: torch.Tensor, group=None, sizes_out=None) -> torch.Tensor:
    """All-gather 1-D uint8 tensors of different lengths; returns the concatenation in rank order
    (the per-rank lengths are appended to ``sizes_out`` when given)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    n = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    if sizes_out is not None:
        sizes_out.extend(sizes)
    m = max(sizes)
    padded = torch.zeros(m, dtype=t.dtype, device=t.device)
    padded[: t.numel()] = t
    outs = [torch.empty(m, dtype=t.dtype, device=t.device) for _ in range(world)]
    dist.all_gather(outs, padded, group=group)
    return torch.cat([o[:s] for o, s in zip(outs, sizes)])


class SlabMergeTree:
    """Context for planes [z_begin, z_end) of an nx x ny x nz grid on one device."""

    def __init__(self, dims, z_begin: int, z_end: int, device=None, wide: bool = False, workspace=None):
        self.dims = tuple(int(d) for d in dims)
        self.z_begin, self.z_end = int(z_begin), int(z_end)
        nx, ny, _ = self.dims
        self.n = nx * ny * (self.z_end - self.z_begin)
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else int(device)) \
            if not isinstance(device, torch.device) else device
        self.device = dev
        nbytes = _lib.mt_slab_workspace_bytes(self.dims, 6, self.z_begin, self.z_end)
        if nbytes == 0:
            raise _lib.MTError(_lib.MT_ERR_INVALID_ARG, "mt_slab_workspace_bytes")
        # a caller may share one workspace between contexts used one after another (tests)
        self.workspace = workspace if workspace is not None else \
            torch.empty(nbytes + 256, dtype=torch.uint8, device=dev)
        if self.workspace.numel() < nbytes + 256:
            raise ValueError("workspace too small")
        ptr = (self.workspace.data_ptr() + 255) // 256 * 256
        self.ctx = _lib.mt_create_slab(self.dims, 6, self.z_begin, self.z_end, dev.index, ptr, nbytes,
                                       _lib.MT_SLAB_WIDE_IDS if wide else 0)
        self._scratch = None
        self._f = None
        self._T = None

    def __del__(self):
        ctx = getattr(self, "ctx", None)
        if ctx is not None and _lib._lib is not None:
            _lib._lib.mt_destroy(ctx)
            self.ctx = None

    def compute_local(self, f_slab: torch.Tensor, split: bool = False, triplets=None, stream=None):
        """Local phase; ``triplets`` (int64, the slab's n values) receives the tile store now and
        the final store from compute_global."""
        if f_slab.dtype != torch.float32 or not f_slab.is_cuda or not f_slab.is_contiguous() or \
                f_slab.numel() != self.n:
            raise ValueError("f_slab must be a float32 CUDA tensor with the slab's nx*ny*(z_end-z_begin) values")
        if triplets is None:
            triplets = torch.empty(self.n, dtype=torch.int64, device=self.device)
        self._f = f_slab  # borrowed by the library until compute_global's work completes
        self._T = triplets
        _lib.mt_compute_local(self.ctx, f_slab.data_ptr(), triplets.data_ptr(),
                              _lib.MT_FLAG_SPLIT_TREE if split else 0, stream)

    def forest(self, stream=None) -> torch.Tensor:
        """The slab's boundary-forest records as a uint8 CUDA tensor (a view into the workspace)."""
        ptr, n = _lib.mt_forest_view(self.ctx, stream)
        if n == 0:
            return torch.empty(0, dtype=torch.uint8, device=self.device)
        off = ptr - self.workspace.data_ptr()
        return self.workspace[off: off + n * RECORD_BYTES]

    def compute_global(self, all_records: torch.Tensor, z_bounds, counts, stream=None) -> torch.Tensor:
        """Global phase into the triplet buffer of compute_local (returned); ``all_records``: every
        slab's records in slab order, ``counts`` of them per slab."""
        n_all = all_records.numel() // RECORD_BYTES
        if sum(counts) != n_all:
            raise ValueError("counts do not add up to the gathered records")
        need = _lib.mt_forest_scratch_bytes(n_all)
        if self._scratch is None or self._scratch.numel() < need + 256:
            self._scratch = torch.empty(need + 256, dtype=torch.uint8, device=self.device)
        sp = (self._scratch.data_ptr() + 255) // 256 * 256
        triplets = self._T
        _lib.mt_compute_global(self.ctx, all_records.data_ptr() if n_all else 0, counts, z_bounds, sp, need,
                               triplets.data_ptr(), stream)
        return triplets

    def triplets64(self, triplets: torch.Tensor, first: int = 0, count: int | None = None, stream=None):
        """(count, 2) int64 tensor (s, v) of 64-bit global ids of triplets[first:first+count]."""
        if count is None:
            count = self.n - first
        out = torch.empty((count, 2), dtype=torch.int64, device=self.device)
        _lib.mt_triplets64(self.ctx, triplets.data_ptr(), first, count, out.data_ptr(), stream)
        return out

    def diagram64(self, stream=None):
        """Synchronises; (records as a PAIR64_DTYPE numpy array, n_pairs, n_essential)."""
        st, npairs, ness = _lib.mt_diagram64(self.ctx, 0, 0, stream)
        if st != _lib.MT_OK:
            raise _lib.MTError(st, "mt_diagram64")
        k = npairs + ness
        out = torch.empty(k * 24, dtype=torch.uint8, device=self.device)
        if k:
            st, _, _ = _lib.mt_diagram64(self.ctx, out.data_ptr(), k, stream)
            if st != _lib.MT_OK:
                raise _lib.MTError(st, "mt_diagram64")
        return out.cpu().numpy().view(_lib.PAIR64_DTYPE), npairs, ness

    def diagram(self, stream=None):
        """Synchronises; (records (k,4) int32, n_pairs, n_essential) of this slab."""
        st, ptr, npairs, ness = _lib.mt_diagram_view(self.ctx, stream)
        if st != _lib.MT_OK:
            raise _lib.MTError(st, "mt_diagram")
        k = npairs + ness
        out = torch.empty((k, 4), dtype=torch.int32, device=self.device)
        if k:
            st, a, b = _lib.mt_diagram(self.ctx, out.data_ptr(), k, stream)
            if st != _lib.MT_OK:
                raise _lib.MTError(st, "mt_diagram")
        return out, npairs, ness


class NcclSlab:
    """A ``mt_create_dist`` context: the rank's slab with the NCCL exchange inside the library."""

    def __init__(self, dims, rank: int, nranks: int, nccl_id: bytes, device=None, wide: bool = False):
        self.dims = tuple(int(d) for d in dims)
        self.z_bounds = slab_bounds(self.dims[2], nranks)
        self.z_begin, self.z_end = self.z_bounds[rank], self.z_bounds[rank + 1]
        nx, ny, _ = self.dims
        self.n = nx * ny * (self.z_end - self.z_begin)
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else int(device)) \
            if not isinstance(device, torch.device) else device
        self.device = dev
        nbytes = _lib.mt_dist_workspace_bytes(self.dims, 6, rank, nranks)
        if nbytes == 0:
            raise _lib.MTError(_lib.MT_ERR_INVALID_ARG, "mt_dist_workspace_bytes")
        self.workspace = torch.empty(nbytes + 256, dtype=torch.uint8, device=dev)
        ptr = (self.workspace.data_ptr() + 255) // 256 * 256
        self.ctx = _lib.mt_create_dist(self.dims, 6, rank, nranks, nccl_id, dev.index, ptr, nbytes,
                                       _lib.MT_SLAB_WIDE_IDS if wide else 0)
        self._f = None

    def __del__(self):
        ctx = getattr(self, "ctx", None)
        if ctx is not None and _lib._lib is not None:
            _lib._lib.mt_destroy(ctx)
            self.ctx = None

    def compute(self, f_slab: torch.Tensor, split: bool = False, triplets=None, stream=None) -> torch.Tensor:
        if f_slab.dtype != torch.float32 or not f_slab.is_cuda or not f_slab.is_contiguous() or \
                f_slab.numel() != self.n:
            raise ValueError("f_slab must be a contiguous float32 CUDA tensor with the slab's values")
        if triplets is None:
            triplets = torch.empty(self.n, dtype=torch.int64, device=self.device)
        self._f = f_slab
        _lib.mt_compute(self.ctx, f_slab.data_ptr(), triplets.data_ptr(),
                        _lib.MT_FLAG_SPLIT_TREE if split else 0, stream)
        return triplets

    diagram = SlabMergeTree.diagram
    diagram64 = SlabMergeTree.diagram64
    triplets64 = SlabMergeTree.triplets64


def broadcast_unique_id(group=None) -> bytes:
    """Rank 0's NCCL unique id (mt_get_unique_id), broadcast over the torch.distributed group."""
    import torch.distributed as dist

    obj = [_lib.mt_get_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


class DistMergeTree:
    """The global grid split into z-slabs over a torch.distributed group, one slab per rank.
    transport "nccl": the library's own NCCL exchange (mt_create_dist); "torch": the three-call
    ABI with the records all-gathered by torch.distributed (any backend, e.g. gloo)."""

    def __init__(self, dims, group=None, device=None, transport: str = "nccl"):
        import torch.distributed as dist

        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.dims = tuple(int(d) for d in dims)
        self.z_bounds = slab_bounds(self.dims[2], self.world)
        zb, ze = self.z_bounds[self.rank], self.z_bounds[self.rank + 1]
        self.transport = transport
        if transport == "nccl":
            self.slab = NcclSlab(self.dims, self.rank, self.world, broadcast_unique_id(group), device)
        elif transport == "torch":
            self.slab = SlabMergeTree(self.dims, zb, ze, device)
        else:
            raise ValueError(transport)
        self.forest_records = 0

    def compute(self, f_slab: torch.Tensor, split: bool = False, triplets=None) -> torch.Tensor:
        if self.transport == "nccl":
            return self.slab.compute(f_slab, split, triplets)
        self.slab.compute_local(f_slab, split, triplets)
        mine = self.slab.forest()
        sizes = []
        everything = allgather_varsize(mine, self.group, sizes)
        self.forest_records = everything.numel() // RECORD_BYTES
        return self.slab.compute_global(everything, self.z_bounds, [b // RECORD_BYTES for b in sizes])

    def diagram(self):
        return self.slab.diagram()


def virtual_compute(f: torch.Tensor, dims, nranks: int, split: bool = False, wide: bool = False):
    """All slabs on ONE device, the all-gather replaced by a concatenation: the device code of
    the multi-GPU path exercised without several GPUs (tests).  Returns (T, diagram records,
    n_pairs, n_essential, gathered records) assembled in the single-GPU order; wide mode: T as
    (n, 2) int64 global (s, v) and the records as a PAIR64_DTYPE array."""
    nx, ny, nz = dims
    zb = slab_bounds(nz, nranks)
    slabs = [SlabMergeTree(dims, zb[r], zb[r + 1], f.device, wide=wide) for r in range(nranks)]
    plane = nx * ny
    for r, s in enumerate(slabs):
        s.compute_local(f[zb[r] * plane: zb[r + 1] * plane].contiguous(), split)
    forests = [s.forest() for s in slabs]
    counts = [x.numel() // RECORD_BYTES for x in forests]
    everything = torch.cat(forests)
    Ts = [s.compute_global(everything, zb, counts) for s in slabs]
    if wide:
        T64 = torch.cat([s.triplets64(T) for s, T in zip(slabs, Ts)])
        diags = [s.diagram64() for s in slabs]
        fin = np.concatenate([d[0][: d[1]] for d in diags])
        ess = np.concatenate([d[0][d[1]:] for d in diags])
        return (T64, np.concatenate([fin, ess]), sum(d[1] for d in diags), sum(d[2] for d in diags),
                everything.numel() // RECORD_BYTES)
    diags = [s.diagram() for s in slabs]
    fin = torch.cat([d[0][: d[1]] for d in diags])
    ess = torch.cat([d[0][d[1]:] for d in diags])
    npairs = sum(d[1] for d in diags)
    ness = sum(d[2] for d in diags)
    return torch.cat(Ts), torch.cat([fin, ess]), npairs, ness, everything.numel() // RECORD_BYTES
