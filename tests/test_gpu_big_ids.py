"""Vertex ids past 2^31 (reading R18: 32-bit ids, n <= 2^32 - 1; PAPER.md:389-396 packs two
32-bit ids into a 64-bit word): a 1536 x 1536 x 1024 grid (2.42e9 vertices) of the c4 white-noise
recipe, so that half of the id space above 2^31 is merged, repaired and emitted by every kernel.
O1 cannot run at this size in a test, so (1) the invariants that hold at any size, on the GPU with
plain torch ops (I1 key order, I2 s = u iff a lower neighbour exists, I3 one root, I4 #pairs =
#strict minima - 1), and (2) exact triplets and diagram records of samples with ids above 2^31
against O4 (the definition by bounded floods), every sample checked.  ~150 GB of device memory:
opt-in with MT_BIG_IDS=1 (its own gpurun call)."""
import os
import resource

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from paper_2301_10838_b200 import _lib, fields  # noqa: E402

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _log(msg):
    print(f"[big ids] {msg} (maxrss {resource.getrusage(resource.RUSAGE_SELF).ru_maxrss >> 20} GB)", flush=True)


@pytest.mark.skipif(os.environ.get("MT_BIG_IDS") != "1", reason="2.4e9-vertex grid: set MT_BIG_IDS=1")
def test_ids_above_2_31():
    dims = (1536, 1536, 1024)
    nx, ny, nz = dims
    n = nx * ny * nz
    assert n > 2 ** 31
    f = fields.white_noise(dims, 4)
    _log(f"field {dims}, n = {n}")
    fd = torch.from_numpy(f).cuda()
    mt = _lib.MergeTree(dims, 6, device=0)
    T = mt.compute(fd)
    rec, npairs, ness = mt.diagram()
    recs = _lib.pairs_to_numpy(rec)
    del rec, mt
    torch.cuda.empty_cache()
    _log(f"computed: {npairs} finite pairs, {ness} essential")
    g = fd.view(nz, ny, nx)
    has_lower = torch.zeros((nz, ny, nx), dtype=torch.bool, device="cuda")
    has_lower[:, :, 1:] |= g[:, :, :-1] <= g[:, :, 1:]
    has_lower[:, :, :-1] |= g[:, :, 1:] < g[:, :, :-1]
    has_lower[:, 1:, :] |= g[:, :-1, :] <= g[:, 1:, :]
    has_lower[:, :-1, :] |= g[:, 1:, :] < g[:, :-1, :]
    has_lower[1:, :, :] |= g[:-1, :, :] <= g[1:, :, :]
    has_lower[:-1, :, :] |= g[1:, :, :] < g[:-1, :, :]
    has_lower = has_lower.view(-1)
    n_min = int((~has_lower).sum().item())
    assert ness == 1 and npairs == n_min - 1, (npairs, ness, n_min)
    s = (T >> 32) & 0xffffffff
    ids = torch.arange(n, device="cuda", dtype=torch.int64)
    is_reg = s == ids
    v = T & 0xffffffff
    root = is_reg & (v == ids)
    bad_i2 = int(((is_reg != has_lower) & ~root).sum().item())
    del has_lower
    n_root = int(root.sum().item())
    fv = fd[v]
    bad_v = int((~(root | (fv < fd) | ((fv == fd) & (v < ids)))).sum().item())
    del fv
    fs = fd[s]
    bad_s = int((~(root | (fs > fd) | ((fs == fd) & (s >= ids)))).sum().item())
    del fs, is_reg
    _log(f"I2 violations {bad_i2}, roots {n_root}, I1 violations {bad_v} / {bad_s}")
    assert bad_i2 == 0 and n_root == 1 and bad_v == 0 and bad_s == 0
    hi_v = int(((v >= 2 ** 31) & ~root).sum().item())
    hi_s = int((s >= 2 ** 31).sum().item())
    _log(f"{hi_v} triplets point at a representative with id >= 2^31, {hi_s} have s >= 2^31")
    assert hi_v > 0 and hi_s > (n - 2 ** 31) // 2   # the upper id range is in use throughout
    # (2) O4 samples above 2^31, levels in the lowest 20 % (white noise percolates near 31 %)
    rng = np.random.default_rng(31)
    q20 = float(np.quantile(f[rng.integers(0, n, 1 << 22)], 0.2))
    h = 2 ** 31                                    # views of the upper half: no gathers of 2^31 ids
    s_hi, v_hi, ids_hi, f_hi = s[h:], v[h:], ids[h:], fd[h:]
    cand_reg = torch.nonzero((s_hi == ids_hi) & (v_hi != ids_hi) & (f_hi <= q20)).view(-1) + h
    cand_br = torch.nonzero((s_hi != ids_hi) & (fd[s_hi] <= q20)).view(-1) + h
    picks = np.concatenate([cand_reg[torch.from_numpy(rng.integers(0, cand_reg.numel(), 48)).cuda()].cpu().numpy(),
                            cand_br[torch.from_numpy(rng.integers(0, cand_br.numel(), 48)).cuda()].cpu().numpy()])
    Ts = T[torch.from_numpy(picks).cuda()].cpu().numpy().view(np.uint64)
    del cand_reg, cand_br, s_hi, v_hi, ids_hi, f_hi, s, v, ids, root, T, fd
    for u, t in zip(picks.tolist(), Ts.tolist()):
        r = oracle.triplet_at(f, dims, 6, u, cap=1 << 23)
        assert r is not None, f"O4 flood of u={u} passed 2^23 vertices"
        assert (r[0] << 32) | r[1] == t, (u, r, divmod(t, 1 << 32))
        if r[0] != u:
            k = int(np.searchsorted(recs["birth_v"][:npairs], u))
            assert recs[k]["birth_v"] == u and recs[k]["death_v"] == r[0]
            assert recs[k]["birth"].tobytes() == f[u].tobytes() and recs[k]["death"].tobytes() == f[r[0]].tobytes()
    _log(f"all {picks.size} samples with ids >= 2^31 equal O4")
