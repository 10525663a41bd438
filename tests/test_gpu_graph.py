"""Explicit graphs on the GPU (mt_create_graph / mt_compute_graph) vs the graph oracle, bit-exact."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from oracle import brute  # noqa: E402
from paper_2301_10838_b200 import _lib  # noqa: E402

pytestmark = pytest.mark.gpu


def er_graph(rng, n, avg_deg):
    m = int(n * avg_deg / 2)
    a = rng.integers(0, n, m)
    b = rng.integers(0, n, m)
    return list(zip(a.tolist(), b.tolist()))   # includes self-loops and duplicates


def check(f, row, col, split=False):
    n = f.size
    g = _lib.GraphMergeTree(n, max(1, col.size), device=0)
    T = g.compute(torch.from_numpy(f).cuda(), torch.from_numpy(row.astype(np.int64)).cuda(),
                  torch.from_numpy(col.astype(np.int32)).cuda(), split=split)
    rec, npairs, ness = g.diagram()
    To, po, npo, neo = oracle.merge_tree_graph(f, row, col, split)
    assert np.array_equal(T.cpu().numpy().view(np.uint64), To)
    assert (npairs, ness) == (npo, neo)
    assert _lib.pairs_to_numpy(rec).tobytes() == po.tobytes()
    return npo, neo


@pytest.mark.parametrize("n,deg", [(1000, 1.5), (20000, 4.0), (100000, 8.0), (50000, 0.8)])
def test_er_graphs(n, deg):
    rng = np.random.default_rng(n)
    row, col = oracle.csr_from_edges(n, er_graph(rng, n, deg))
    for kind in range(2):
        f = rng.random(n).astype(np.float32) if kind == 0 else rng.integers(0, 7, n).astype(np.float32)
        npo, neo = check(f, row, col, split=bool(kind))
    assert neo >= 1


def test_grid_as_graph_on_gpu():
    dims = (40, 30, 20)
    n = 40 * 30 * 20
    f = np.random.default_rng(5).random(n).astype(np.float32)
    edges = [(u, w) for u in range(n) for w in brute.grid_neighbours(u, dims) if w > u]
    row, col = oracle.csr_from_edges(n, edges)
    check(f, row, col)


def test_edgeless_and_tiny():
    for n in (1, 2, 7):
        row, col = oracle.csr_from_edges(n, [])
        check(np.arange(n, dtype=np.float32)[::-1].copy(), row, col)


def test_adjacency_longer_than_context_is_reported():
    """row[n] > n_adj through the raw C ABI: MT_ERR_CAPACITY at mt_diagram, never a silently
    wrong tree (the queue would drop edges)."""
    n = 2000
    rng = np.random.default_rng(7)
    row, col = oracle.csr_from_edges(n, er_graph(rng, n, 6.0))
    small = 100
    nbytes = _lib.mt_graph_workspace_bytes(n, small)
    ws = torch.empty(nbytes + 256, dtype=torch.uint8, device="cuda")
    ctx = _lib.mt_create_graph(n, small, 0, (ws.data_ptr() + 255) // 256 * 256, nbytes)
    try:
        f = torch.from_numpy(rng.random(n).astype(np.float32)).cuda()
        r = torch.from_numpy(row.astype(np.int64)).cuda()
        c = torch.from_numpy(col.astype(np.int32)).cuda()
        T = torch.empty(n, dtype=torch.int64, device="cuda")
        _lib.mt_compute_graph(ctx, f.data_ptr(), r.data_ptr(), c.data_ptr(), T.data_ptr())
        st, _, _ = _lib.mt_diagram(ctx)
        assert st == _lib.MT_ERR_CAPACITY
    finally:
        _lib.mt_destroy(ctx)


def test_graph_compute_rejects_wrong_dtypes():
    n = 10
    row, col = oracle.csr_from_edges(n, [(i, i + 1) for i in range(n - 1)])
    g = _lib.GraphMergeTree(n, col.size, device=0)
    f = torch.zeros(n, dtype=torch.float32, device="cuda")
    r = torch.from_numpy(row.astype(np.int64)).cuda()
    with pytest.raises(ValueError):
        g.compute(f, r, torch.from_numpy(col.astype(np.int64)).cuda())
    with pytest.raises(ValueError):
        g.compute(f.double(), r, torch.from_numpy(col.astype(np.int32)).cuda())
