"""Diagnostics: per-kernel times and merge/repair event counters for each config."""
import json
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2301_10838_b200 import _lib, fields

cfgs = sys.argv[1:] or ["c2", "c3", "c4", "c5"]
for cfg in cfgs:
    f, dims, conn = fields.make(cfg, device="cuda" if cfg == "c5" else "cpu")
    n = int(np.prod(dims))
    mt = _lib.MergeTree(dims, conn, device=0)
    fd = torch.from_numpy(f).cuda()
    T = torch.empty(n, dtype=torch.int64, device="cuda")
    for _ in range(2):
        _lib.mt_compute(mt.ctx, fd.data_ptr(), T.data_ptr(), 0)
        _lib.mt_diagram(mt.ctx)
    _lib.mt_set_profiling(mt.ctx, True)
    _lib.mt_compute(mt.ctx, fd.data_ptr(), T.data_ptr(), 0)
    st, npairs, ness = _lib.mt_diagram(mt.ctx)
    times = _lib.mt_kernel_times(mt.ctx)
    _lib.mt_set_profiling(mt.ctx, False)
    _lib.mt_set_stats(mt.ctx, True)
    _lib.mt_compute(mt.ctx, fd.data_ptr(), T.data_ptr(), 0)
    _lib.mt_diagram(mt.ctx)
    stats = _lib.mt_stats(mt.ctx)
    _lib.mt_set_stats(mt.ctx, False)
    per = {k: v / n for k, v in stats.items()}
    print(json.dumps({"cfg": cfg, "n": n, "pairs": npairs, "times_ms": times, "stats": stats,
                      "per_vertex": per}), flush=True)
    del mt, fd, T
    torch.cuda.empty_cache()
