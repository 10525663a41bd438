"""Multi-GPU estimate on ONE GPU: the z-slab path of P ranks run as P virtual ranks one after the
other (the NCCL all-gather replaced by a concatenation), each phase timed with CUDA events.
Per-rank step estimate = max local + all-gather (records x P over NVLink at a stated rate) +
max global.  An estimate, not a measurement of P GPUs."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2301_10838_b200 import fields
from paper_2301_10838_b200.dist import SlabMergeTree, slab_bounds

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
Ps = [int(p) for p in sys.argv[2:]] or [2, 4, 8]
f, dims, _ = fields.make(cfg, device="cuda" if cfg == "c5" else "cpu")
fd = torch.from_numpy(f).cuda()
nx, ny, nz = dims
NVLINK_GBPS = 770.0   # per-direction peer copy MEASURED on this pool (B200_PROFILING.md; 900 nominal)


def timed(fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


for P in Ps:
    zb = slab_bounds(nz, P)
    slabs = [SlabMergeTree(dims, zb[r], zb[r + 1]) for r in range(P)]
    parts = [fd[zb[r] * nx * ny: zb[r + 1] * nx * ny].contiguous() for r in range(P)]
    best_loc, best_glob = [1e30] * P, [1e30] * P
    for rep in range(5):   # per rank, the best of the last four passes
        loc = [timed(lambda r=r: slabs[r].compute_local(parts[r])) for r in range(P)]
        recs = [s.forest() for s in slabs]
        counts = [x.numel() // 32 for x in recs]
        allr = torch.cat(recs)
        glob = [timed(lambda r=r: slabs[r].compute_global(allr, zb, counts)) for r in range(P)]
        if rep:
            best_loc = [min(a, b) for a, b in zip(best_loc, loc)]
            best_glob = [min(a, b) for a, b in zip(best_glob, glob)]
    loc, glob = best_loc, best_glob
    # per-kernel split of one rank (library profiling marks)
    from paper_2301_10838_b200 import _lib
    _lib.mt_set_profiling(slabs[-1].ctx, True)
    slabs[-1].compute_local(parts[-1])
    slabs[-1].compute_global(allr, zb, counts)
    torch.cuda.synchronize()
    split = _lib.mt_kernel_times(slabs[-1].ctx)
    _lib.mt_set_profiling(slabs[-1].ctx, False)
    gather_ms = allr.numel() / 1e9 / NVLINK_GBPS * 1e3
    est = max(loc) + gather_ms + max(glob)
    print(json.dumps({"cfg": cfg, "P": P, "local_ms_max": max(loc), "local_ms": loc, "global_ms_max": max(glob),
                      "global_ms": glob, "forest_bytes_all": allr.numel(), "allgather_ms_est": gather_ms,
                      "step_ms_est": est, "Mv_s_est": nx * ny * nz / est / 1e3,
                      "assumed_allgather_GBps": NVLINK_GBPS,
                      "last_rank_kernels_ms": split}), flush=True)
    del slabs, parts, recs, allr
    torch.cuda.empty_cache()
