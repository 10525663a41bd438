"""Step-by-step virtual-rank run with syncs and prints (locates a hang or mismatch)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2301_10838_b200 import _lib, fields
from paper_2301_10838_b200.dist import SlabMergeTree, slab_bounds

cfg, scale, P = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
f, dims, _ = fields.make(cfg, scale=scale)
fd = torch.from_numpy(f).cuda()
nx, ny, nz = dims
zb = slab_bounds(nz, P)
print("bounds", zb, flush=True)
slabs = [SlabMergeTree(dims, zb[r], zb[r + 1]) for r in range(P)]
for r, s in enumerate(slabs):
    s.compute_local(fd[zb[r] * nx * ny: zb[r + 1] * nx * ny].contiguous())
    torch.cuda.synchronize()
    print("local", r, "forest", s.forest().numel() // 32, flush=True)
recs = [s.forest() for s in slabs]
counts = [x.numel() // 32 for x in recs]
allr = torch.cat(recs)
for r, s in enumerate(slabs):
    t = time.time()
    s.compute_global(allr, zb, counts)
    torch.cuda.synchronize()
    st = _lib.mt_last_error(s.ctx)
    print("global", r, "status", st, round(time.time() - t, 3), flush=True)
