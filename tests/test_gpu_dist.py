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


def test_nccl_dist_one_rank_wide_ids():
    """mt_create_dist with MT_SLAB_WIDE_IDS: the rank's view and the 64-bit translation through
    the library's own exchange path (one rank: every id is the rank's own)."""
    from paper_2301_10838_b200.dist import NcclSlab
    f, dims, _ = fields.make("c4", scale=40)
    s = NcclSlab(dims, 0, 1, _lib.mt_get_unique_id(), device=0, wide=True)
    T = s.compute(torch.from_numpy(f).cuda())
    T64 = s.triplets64(T).cpu().numpy().view(np.uint64)
    rec64, npairs, ness = s.diagram64()
    To, po, npo, neo = oracle.merge_tree(f, dims, conn=6)
    assert np.array_equal(T64[:, 0], To >> np.uint64(32)) and np.array_equal(T64[:, 1], To & np.uint64(0xffffffff))
    assert (npairs, ness) == (npo, neo)
    assert np.array_equal(rec64["death_v"], po["death_v"].astype(np.uint64))


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


# ---- wide ids: the same parity with every slab working in its own
# 32-bit view (compressed ids of the other slabs, 64-bit decode), forced at sizes O1 can check;
# tests/test_gpu_f3_big.py runs a grid past 2^32 vertices.

def check_wide(f, dims, nranks, split=False):
    T64, rec64, npairs, ness, nrec = virtual_compute(torch.from_numpy(f).cuda(), dims, nranks, split, wide=True)
    To, po, npo, neo = oracle.merge_tree(f, dims, conn=6, split=split)
    T64 = T64.cpu().numpy().view(np.uint64).reshape(-1, 2)
    s_o, v_o = To >> np.uint64(32), To & np.uint64(0xffffffff)
    bad = np.nonzero((T64[:, 0] != s_o) | (T64[:, 1] != v_o))[0]
    if bad.size:
        u = int(bad[0])
        raise AssertionError(f"wide P={nranks}: {bad.size} triplets differ; first u={u}: gpu {tuple(T64[u])} "
                             f"oracle ({s_o[u]}, {v_o[u]})")
    assert (npairs, ness) == (npo, neo)
    assert np.array_equal(rec64["birth_v"], po["birth_v"].astype(np.uint64))
    assert np.array_equal(rec64["death_v"], po["death_v"].astype(np.uint64))
    assert rec64["birth"].tobytes() == po["birth"].tobytes() and rec64["death"].tobytes() == po["death"].tobytes()
    return nrec


@pytest.mark.parametrize("nranks", [2, 3, 4, 8])
def test_wide_ids_virtual_ranks_white_noise(nranks):
    f, dims, _ = fields.make("c4", scale=64)
    check_wide(f, dims, nranks)
    check_wide(f, dims, nranks, split=True)


@pytest.mark.parametrize("cfg,scale,nranks", [("c5", 96, 5), ("c3", 64, 2), ("c1", 16, 16), ("c4", 48, 3)])
def test_wide_ids_virtual_ranks_recipes(cfg, scale, nranks):
    f, dims, _ = fields.make(cfg, scale=scale)
    check_wide(f, dims, nranks)


@pytest.mark.parametrize("dims,nranks", [((33, 9, 17), 3), ((40, 40, 5), 5), ((7, 300, 9), 2)])
def test_wide_ids_virtual_ranks_ragged_and_ties(dims, nranks):
    rng = np.random.default_rng(sum(dims) + 1)
    n = int(np.prod(dims))
    for f in (rng.random(n).astype(np.float32), rng.integers(0, 4, n).astype(np.float32)):
        check_wide(f, dims, nranks)
    check_wide(np.full(n, 2.5, np.float32), dims, nranks)                   # id order only


def test_wide_ids_zero_saddles_and_32bit_calls_refused():
    dims = (40, 24, 32)
    z, y, x = np.meshgrid(np.arange(32), np.arange(24), np.arange(40), indexing="ij")
    rng = np.random.default_rng(12)
    f = np.where((x + y + z) % 2 == 0, -1.0, 0.0).astype(np.float32)
    f[(f == 0.0) & (rng.random(f.shape) < 0.5)] = -0.0
    check_wide(f.reshape(-1), dims, 4)
    from paper_2301_10838_b200.dist import SlabMergeTree, slab_bounds
    zb = slab_bounds(32, 2)
    s = SlabMergeTree(dims, zb[0], zb[1], wide=True)
    s.compute_local(torch.from_numpy(f.reshape(-1)[: s.n].copy()).cuda())
    out = torch.empty(16, dtype=torch.int64, device="cuda")
    with pytest.raises(_lib.MTError):      # before the global phase there is no id translation
        s.triplets64(s._T, 0, 1)
    st, _, _ = _lib.mt_diagram(s.ctx, out.data_ptr(), 1)
    assert st == _lib.MT_ERR_TOO_LARGE     # view ids never leave through the 32-bit calls


def test_triplets64_on_one_gpu_widens():
    """mt_triplets64 / mt_diagram64 on a single-GPU context: the 32-bit result widened."""
    f, dims, conn = fields.make("c1")
    mt = _lib.MergeTree(dims, conn, device=0)
    T = mt.compute(torch.from_numpy(f).cuda())
    out = torch.empty((T.numel(), 2), dtype=torch.int64, device="cuda")
    _lib.mt_triplets64(mt.ctx, T.data_ptr(), 0, T.numel(), out.data_ptr())
    Tn = T.cpu().numpy().view(np.uint64)
    o = out.cpu().numpy().view(np.uint64)
    assert np.array_equal(o[:, 0], Tn >> np.uint64(32)) and np.array_equal(o[:, 1], Tn & np.uint64(0xffffffff))
    st, npairs, ness = _lib.mt_diagram64(mt.ctx, 0, 0)
    buf = torch.empty((npairs + ness) * 24, dtype=torch.uint8, device="cuda")
    st, _, _ = _lib.mt_diagram64(mt.ctx, buf.data_ptr(), npairs + ness)
    assert st == _lib.MT_OK
    r64 = buf.cpu().numpy().view(_lib.PAIR64_DTYPE)
    rec, a, b = mt.diagram()
    r32 = _lib.pairs_to_numpy(rec)
    assert np.array_equal(r64["birth_v"], r32["birth_v"].astype(np.uint64))
    assert np.array_equal(r64["death_v"], r32["death_v"].astype(np.uint64))
