"""Multi-GPU path on one GPU ("virtual ranks"): every slab's device code (local merge tree,
boundary forest, forest merge, write-back, repair with remote lookups) runs for P slabs on
cuda:0 with the all-gather replaced by a concatenation; the assembled triplets and diagram
must equal the oracle bit for bit (and therefore the single-GPU result)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from paper_2301_10838_b200 import _lib, fields  # noqa: E402
from paper_2301_10838_b200.dist import virtual_compute  # noqa: E402

pytestmark = pytest.mark.gpu


def check(f, dims, nranks, split=False):
    T, rec, npairs, ness, nrec = virtual_compute(torch.from_numpy(f).cuda(), dims, nranks, split)
    To, po, npo, neo = oracle.merge_tree(f, dims, conn=6, split=split)
    T = T.cpu().numpy().view(np.uint64)
    if not np.array_equal(T, To):
        bad = np.nonzero(T != To)[0]
        u = int(bad[0])
        raise AssertionError(f"P={nranks}: {bad.size} cells differ; first u={u}: gpu (s={T[u] >> 32}, "
                             f"v={T[u] & 0xffffffff}) oracle (s={To[u] >> 32}, v={To[u] & 0xffffffff})")
    assert (npairs, ness) == (npo, neo)
    assert _lib.pairs_to_numpy(rec).tobytes() == po.tobytes()
    return nrec


@pytest.mark.parametrize("nranks", [2, 3, 4, 8])
def test_virtual_ranks_white_noise(nranks):
    f, dims, _ = fields.make("c4", scale=64)
    check(f, dims, nranks)
    check(f, dims, nranks, split=True)


@pytest.mark.parametrize("cfg,scale,nranks", [("c5", 96, 5), ("c3", 64, 2), ("c1", 16, 16), ("c4", 48, 3)])
def test_virtual_ranks_recipes(cfg, scale, nranks):
    f, dims, _ = fields.make(cfg, scale=scale)
    check(f, dims, nranks)


@pytest.mark.parametrize("dims,nranks", [((33, 9, 17), 3), ((40, 40, 5), 5), ((7, 300, 9), 2)])
def test_virtual_ranks_ragged(dims, nranks):
    rng = np.random.default_rng(sum(dims))
    n = int(np.prod(dims))
    for f in (rng.random(n).astype(np.float32), rng.integers(0, 4, n).astype(np.float32)):
        check(f, dims, nranks)


def test_virtual_ranks_closed_forms():
    dims = (24, 20, 16)
    z, y, x = np.meshgrid(np.arange(16), np.arange(20), np.arange(24), indexing="ij")
    check(((x + y + z) % 2).astype(np.float32).reshape(-1), dims, 4)     # 50% minima
    check(np.full(24 * 20 * 16, 1.5, np.float32), dims, 4)               # id order only


@pytest.mark.parametrize("cfg,scale,split", [("c4", 48, False), ("c5", 64, True)])
def test_nccl_dist_one_rank_through_c_abi(cfg, scale, split):
    """mt_get_unique_id + mt_create_dist with a 1-rank NCCL communicator (one GPU per box here),
    then mt_compute / mt_diagram exactly as on one GPU: the library's own exchange path (NCCL
    all-gather of the forest size, grouped broadcasts of the records, global phase) must give
    the oracle's store and diagram bit for bit."""
    from paper_2301_10838_b200.dist import NcclSlab
    f, dims, _ = fields.make(cfg, scale=scale)
    s = NcclSlab(dims, 0, 1, _lib.mt_get_unique_id(), device=0)
    for _ in range(2):   # the second step reuses the grown exchange buffers
        T = s.compute(torch.from_numpy(f).cuda(), split=split)
        rec, npairs, ness = s.diagram()
        To, po, npo, neo = oracle.merge_tree(f, dims, conn=6, split=split)
        assert np.array_equal(T.cpu().numpy().view(np.uint64), To)
        assert (npairs, ness) == (npo, neo)
        assert _lib.pairs_to_numpy(rec).tobytes() == po.tobytes()
    assert _lib.mt_last_launch_count(s.ctx) >= 6


def test_virtual_ranks_zero_saddles():
    """Saddles at -0.0 / +0.0 across slab boundaries: the diagram's death values are the input's
    bits (reading R14) even when the saddle's record lives on another rank (the forest keeps the f
    bits of zero-valued saddles, whose order key cannot tell -0 from +0, reading R2)."""
    dims = (40, 24, 32)
    z, y, x = np.meshgrid(np.arange(32), np.arange(24), np.arange(40), indexing="ij")
    rng = np.random.default_rng(11)
    f = np.where((x + y + z) % 2 == 0, -1.0, 0.0).astype(np.float32)
    neg = rng.random(f.shape) < 0.5
    f[(f == 0.0) & neg] = -0.0
    f = f.reshape(-1)
    for p in (2, 4):
        check(f, dims, p)
