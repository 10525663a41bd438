"""Small end-to-end runs for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
from paper_2301_10838_b200 import _lib, fields
from paper_2301_10838_b200.dist import virtual_compute

ok = True
for cfg, scale in [("c4", 40), ("c5", 48), ("c2", 80)]:
    f, dims, conn = fields.make(cfg, scale=scale)
    mt = _lib.MergeTree(dims, conn, device=0)
    T = mt.compute(torch.from_numpy(f).cuda())
    rec, a, b = mt.diagram()
    To, po, npo, neo = oracle.merge_tree(f, dims, conn)
    ok &= bool(np.array_equal(T.cpu().numpy().view(np.uint64), To))
    mt.filter_diagram(0.01)
f, dims, conn = fields.make("c4", scale=32)
T, rec, a, b, nrec = virtual_compute(torch.from_numpy(f).cuda(), dims, 3)
To, po, npo, neo = oracle.merge_tree(f, dims, conn)
ok &= bool(np.array_equal(T.cpu().numpy().view(np.uint64), To))
print("parity", ok)
