"""GPU parity: the CUDA path (through the C ABI) vs the oracle O1, bit-exact.

The triplet store is unique for the (value, id) order, so the
uint64 cells and the ordered diagram records (birth_v, death_v, f bits) are
compared with memcmp semantics.  Sizes: golden fixtures, 100 seeds of the c1
config, ragged shapes that span several tiles with partial tails, every
BASELINE config scaled down, closed-form stress families, and the full-size
configs c2/c3/c4 in the launch configuration bench.py times.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from oracle import invariants  # noqa: E402
from paper_2301_10838_b200 import _lib, fields  # noqa: E402
from golden_io import all_cases  # noqa: E402

pytestmark = pytest.mark.gpu

_CTX = {}


def ctx_for(dims, conn):
    key = (tuple(dims), conn)
    if key not in _CTX:
        if len(_CTX) > 8:
            _CTX.clear()
        _CTX[key] = _lib.MergeTree(dims, conn, device=0)
    return _CTX[key]


def gpu_tree(f, dims, conn, split=False):
    mt = ctx_for(dims, conn)
    fd = torch.from_numpy(np.ascontiguousarray(f, dtype=np.float32)).cuda()
    T = mt.compute(fd, split=split)
    rec, npairs, ness = mt.diagram()
    return T.cpu().numpy().view(np.uint64), _lib.pairs_to_numpy(rec), npairs, ness


def assert_parity(f, dims, conn, split=False, check_invariants=False):
    T, pairs, npairs, ness = gpu_tree(f, dims, conn, split)
    To, po, npo, neo = oracle.merge_tree(f, dims, conn=conn, split=split)
    if not np.array_equal(T, To):
        bad = np.nonzero(T != To)[0]
        u = int(bad[0])
        raise AssertionError(f"{bad.size} cells differ; first u={u}: gpu (s={T[u] >> 32}, v={T[u] & 0xffffffff}) "
                             f"oracle (s={To[u] >> 32}, v={To[u] & 0xffffffff})")
    assert (npairs, ness) == (npo, neo)
    assert pairs.tobytes() == po.tobytes()
    if check_invariants:
        invariants.check(T, f, dims, split=split, n_pairs=npairs, n_ess=ness)
    return npairs


@pytest.mark.parametrize("case", all_cases(), ids=lambda c: c["name"])
def test_golden_on_gpu(case):
    assert_parity(case["f"], case["dims"], case["conn"], case["split"])


def test_c1_hundred_seeds():
    """c1 recipe (16^3 u24 white noise, 6-conn), parity seeds 0-99."""
    for seed in range(100):
        f = fields.white_noise((16, 16, 16), seed)
        assert_parity(f, (16, 16, 16), 6, split=bool(seed % 2))


@pytest.mark.parametrize("dims", [(33, 9, 17), (1, 1, 1000), (1000, 1, 1), (7, 300, 1), (65, 66, 3),
                                  (2, 2, 2), (31, 1, 9), (100, 100, 1), (45, 37, 29)])
def test_ragged_shapes(dims):
    rng = np.random.default_rng(sum(dims))
    n = int(np.prod(dims))
    conn = 4 if dims[2] == 1 else 6
    for kind in range(3):
        if kind == 0:
            f = rng.random(n).astype(np.float32)
        elif kind == 1:
            f = rng.integers(0, 5, n).astype(np.float32)          # heavy ties
        else:
            f = np.where(rng.random(n) < 0.5, -0.0, 0.0).astype(np.float32)  # all-equal values, +-0
        assert_parity(f, dims, conn, split=bool(kind == 1), check_invariants=True)


@pytest.mark.parametrize("cfg,scale", [("c2", 512), ("c3", 64), ("c4", 96), ("c1", 40), ("c2", 97)])
def test_scaled_configs(cfg, scale):
    f, dims, conn = fields.make(cfg, scale=scale)
    assert_parity(f, dims, conn, check_invariants=True)
    assert_parity(f, dims, conn, split=True)


@pytest.mark.parametrize("dims", [(64, 64, 64), (256, 256, 1)])
def test_closed_form_stress(dims):
    nx, ny, nz = dims
    conn = 4 if nz == 1 else 6
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    checker = ((x + y + z) % 2).astype(np.float32).reshape(-1)   # 50% minima: CAS contention
    npairs = assert_parity(checker, dims, conn)
    assert npairs == int((checker == 0).sum()) - 1
    const = np.full(nx * ny * nz, 3.0, np.float32)               # id order only
    assert assert_parity(const, dims, conn) == 0
    ramp = (x + y + z).astype(np.float32).reshape(-1)
    assert assert_parity(-ramp, dims, conn) == 0


@pytest.mark.parametrize("dims", [(64, 64, 64), (96, 40, 1), (40, 7, 3)])
def test_repair_long_walks(dims):
    """Checkerboard + noise (every vertex pair of basins adjacent, long repair walks): parity,
    and the repair walked cells."""
    nx, ny, nz = dims
    conn = 4 if nz == 1 else 6
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    checker = ((x + y + z) % 2).astype(np.float32).reshape(-1)
    checker += np.random.default_rng(5).random(checker.size).astype(np.float32) * 0.5   # distinct saddles
    mt = _lib.MergeTree(dims, conn, device=0)
    _lib.mt_set_stats(mt.ctx, True)
    T = mt.compute(torch.from_numpy(checker).cuda())
    rec, npairs, ness = mt.diagram()
    st = _lib.mt_stats(mt.ctx)
    To, po, npo, neo = oracle.merge_tree(checker, dims, conn=conn)
    assert np.array_equal(T.cpu().numpy().view(np.uint64), To)
    assert _lib.pairs_to_numpy(rec).tobytes() == po.tobytes()
    assert st["repair_hops"] > 0


def test_empty_and_single():
    for dims in [(0, 5, 5), (5, 0, 1)]:
        mt = _lib.MergeTree(dims, 6 if dims[2] > 1 else 4, device=0)
        f = torch.empty(0, dtype=torch.float32, device="cuda")
        T = mt.compute(f)
        rec, npairs, ness = mt.diagram()
        assert T.numel() == 0 and npairs == 0 and ness == 0
    assert_parity(np.array([4.0], np.float32), (1, 1, 1), 6)


def test_nonfinite_is_reported():
    f = fields.white_noise((20, 20, 20), 3)
    for bad in (np.nan, np.inf, -np.inf):
        g = f.copy()
        g[4321] = bad
        mt = ctx_for((20, 20, 20), 6)
        mt.compute(torch.from_numpy(g).cuda())
        st, _, _ = _lib.mt_diagram(mt.ctx)
        assert st == _lib.MT_ERR_NONFINITE
    # the context recovers on the next valid input
    assert_parity(f, (20, 20, 20), 6)


def test_registered_output_and_capacity():
    f, dims, conn = fields.make("c4", scale=40)
    To, po, npo, neo = oracle.merge_tree(f, dims, conn)
    mt = _lib.MergeTree(dims, conn, device=0)
    fd = torch.from_numpy(f).cuda()
    buf = torch.zeros((npo + neo, 4), dtype=torch.int32, device="cuda")
    mt.set_diagram_output(buf)
    mt.compute(fd)
    st, a, b = _lib.mt_diagram(mt.ctx, buf.data_ptr(), buf.shape[0])
    assert st == _lib.MT_OK and (a, b) == (npo, neo)
    assert _lib.pairs_to_numpy(buf).tobytes() == po.tobytes()
    small = torch.zeros((npo // 2, 4), dtype=torch.int32, device="cuda")
    mt.set_diagram_output(small)
    mt.compute(fd)
    st, a, b = _lib.mt_diagram(mt.ctx)
    assert st == _lib.MT_ERR_CAPACITY and (a, b) == (npo, neo)   # required counts still reported


def test_repeat_runs_identical():
    f, dims, conn = fields.make("c4", scale=128)
    mt = ctx_for(dims, conn)
    fd = torch.from_numpy(f).cuda()
    first = mt.compute(fd).clone()
    rec0, _, _ = mt.diagram()
    for _ in range(5):
        assert torch.equal(mt.compute(fd), first)
        rec, _, _ = mt.diagram()
        assert torch.equal(rec, rec0)


def test_launches_are_library_kernels():
    f, dims, conn = fields.make("c1")
    mt = ctx_for(dims, conn)
    mt.compute(torch.from_numpy(f).cuda())
    mt.diagram()
    assert mt.last_launch_count() == 6


@pytest.mark.parametrize("cfg", ["c2", "c3", "c4"])
def test_full_size_configs(cfg):
    """BASELINE configs at full size, same launch configuration as bench.py, bit-exact vs O1."""
    f, dims, conn = fields.make(cfg)
    assert_parity(f, dims, conn, check_invariants=(cfg != "c4"))


@pytest.mark.parametrize("cfg", ["c4", "c5", "c3"])
def test_medium_many_seeds(cfg):
    """Concurrency stress at 128^3: many seeds of the noise / GRF / smooth recipes."""
    for seed in range(6):
        f, dims, conn = fields.make(cfg, seed=100 + seed, scale=128)
        assert_parity(f, dims, conn, split=bool(seed % 2))


@pytest.mark.parametrize("cfg,scale,split", [("c4", 64, False), ("c5", 64, True), ("c2", 256, False)])
def test_persistence_filter(cfg, scale, split):
    """mt_filter_diagram == the oracle's filter of the oracle diagram, order preserved."""
    f, dims, conn = fields.make(cfg, scale=scale)
    To, po, npo, neo = oracle.merge_tree(f, dims, conn=conn, split=split)
    mt = ctx_for(dims, conn)
    mt.compute(torch.from_numpy(f).cuda(), split=split)
    pers = np.abs(po["death"][:npo] - po["birth"][:npo])
    for eps in (0.0, float(np.quantile(pers, 0.5)) if npo else 0.1, float(pers.max()) if npo else 1.0, 1e30):
        rec, a, b = mt.filter_diagram(eps)
        want = oracle.filter_by_persistence(po, npo, eps)
        assert a + b == want.size and b == neo
        assert _lib.pairs_to_numpy(rec).tobytes() == want.tobytes()


def test_host_pipeline_outputs():
    """The overlapped host->host pipeline returns, for every field, exactly the oracle's store
    and diagram (double buffers must not mix steps)."""
    from paper_2301_10838_b200.pipeline import HostPipeline
    dims = (48, 40, 36)
    fs = [fields.white_noise(dims, 50 + i) for i in range(4)]
    pipe = HostPipeline(dims, 6, device=0)
    n = int(np.prod(dims))
    f_hosts = [torch.from_numpy(f).pin_memory() for f in fs]
    T_hosts = [torch.empty(n, dtype=torch.int64).pin_memory() for _ in fs]
    rec_hosts = [torch.empty((n // 2 + 2, 4), dtype=torch.int32).pin_memory() for _ in fs]
    counts = pipe.run(f_hosts, T_hosts, rec_hosts)
    for f, T, rec, (a, b) in zip(fs, T_hosts, rec_hosts, counts):
        To, po, npo, neo = oracle.merge_tree(f, dims, 6)
        assert np.array_equal(T.numpy().view(np.uint64), To)
        assert (a, b) == (npo, neo)
        assert rec[: a + b].numpy().view(_lib.PAIR_DTYPE).reshape(-1).tobytes() == po.tobytes()


def test_full_size_c5_sampled():
    """c5 at its full 1024^3 size in bench.py's launch configuration (the full O1 memcmp is
    tests/test_gpu_full_c5.py, opt-in): (1) properties that hold at any size, computed
    independently on the GPU with plain torch ops: I1 key(v) < key(u) <= key(s) for non-roots,
    I2 s = u iff u has a lower neighbour, I3 one root, I4 #finite pairs = #strict local minima - 1;
    (2) exact triplets and diagram records of level-stratified samples against O4 (the definition
    by bounded floods, oracle.triplet_at), every sample checked."""
    import resource
    log = lambda msg: print(f"[c5] {msg}: maxrss {resource.getrusage(resource.RUSAGE_SELF).ru_maxrss >> 20} GB",
                            flush=True)
    f, dims, conn = fields.make("c5", device="cuda")
    log("field")
    nx, ny, nz = dims
    n = nx * ny * nz
    fd = torch.from_numpy(f).cuda()
    mt = _lib.MergeTree(dims, conn, device=0)
    T = mt.compute(fd)
    rec, npairs, ness = mt.diagram()
    torch.cuda.synchronize()
    log("computed")
    # (1) invariants, on the GPU with torch (ties broken by id: a lower-id neighbour is lower
    # when equal, reading R1; -0.0 == +0.0 under float compares, reading R2)
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
    v = T & 0xffffffff
    ids = torch.arange(n, device="cuda", dtype=torch.int64)
    is_reg = s == ids
    root = is_reg & (v == ids)
    bad_i2 = int(((is_reg != has_lower) & ~root).sum().item())    # I2 is about non-root cells
    del has_lower
    n_root = int(root.sum().item())
    fv = fd[v]
    bad_v = int((~(root | (fv < fd) | ((fv == fd) & (v < ids)))).sum().item())
    del fv
    fs = fd[s]
    bad_s = int((~(root | (fs > fd) | ((fs == fd) & (s >= ids)))).sum().item())
    del fs, root, ids, is_reg
    log(f"I2 violations {bad_i2}, roots {n_root}, I1 violations {bad_v} / {bad_s}")
    assert bad_i2 == 0, "I2: s = u exactly at the non-root vertices with a lower neighbour"
    assert n_root == 1, "I3: one root"
    assert bad_v == 0 and bad_s == 0, "I1: key(v) < key(u) <= key(s)"
    log("invariants")
    # (2) exact triplets (O4) of samples stratified by level, none skipped.  O4 floods the
    # sublevel component of u, so it can only reach levels below 3-D percolation (the first run,
    # gpurun_out r2a, saw a flood past 2^23 vertices in the 15-20 % stratum: this field's sublevel
    # sets percolate there): regular vertices are stratified by their own level over the lowest
    # 12 % (4 strata of 3 %), branches (minima) by their death level over the same range,
    # 12 samples per stratum.
    # Every sample must be checked: a flood past the cap FAILS the test (a wrong, too-low saddle
    # from the GPU would otherwise be skipped).  Vertices above percolation are covered by the
    # invariants above and by the full O1 memcmp (tests/test_gpu_full_c5.py, MT_FULL_C5=1).
    rng = np.random.default_rng(2301)
    ids = torch.arange(n, device="cuda", dtype=torch.int64)
    is_branch = s != ids
    lev_u = fd
    lev_d = fd[s]
    qs = torch.quantile(fd[torch.from_numpy(rng.integers(0, n, 1 << 23)).cuda()],
                        torch.tensor([0.0, 0.03, 0.06, 0.09, 0.12], device="cuda")).tolist()
    qs[0] = -float("inf")
    picks, labels = [], []
    for kind, mask, lev in (("regular", ~is_branch & (v != ids), lev_u), ("branch", is_branch, lev_d)):
        for j in range(4):
            cand = torch.nonzero(mask & (lev > qs[j]) & (lev <= qs[j + 1]), as_tuple=False).view(-1)
            assert cand.numel() >= 12, (kind, j, cand.numel())
            sel = cand[torch.from_numpy(rng.integers(0, cand.numel(), 12)).cuda()].cpu().numpy()
            picks.extend(sel.tolist())
            labels.extend([f"{kind} level q{3 * j}-{3 * j + 3}%"] * sel.size)
            del cand
    del ids, is_branch, lev_d
    picks = np.asarray(picks, dtype=np.int64)
    Ts = T[torch.from_numpy(picks).cuda()].cpu().numpy().view(np.uint64)
    recs = _lib.pairs_to_numpy(rec)
    log("samples")
    checked = {}
    for u, t, lab in zip(picks.tolist(), Ts.tolist(), labels):
        r = oracle.triplet_at(f, dims, conn, u, cap=1 << 23)
        assert r is not None, f"O4 flood of sample u={u} ({lab}) passed 2^23 vertices"
        assert (r[0] << 32) | r[1] == t, (u, lab, r, divmod(t, 1 << 32))
        if r[0] != u:   # a branch born at u dies at s: its record, in ascending-birth order
            k = int(np.searchsorted(recs["birth_v"][:npairs], u))
            assert recs[k]["birth_v"] == u and recs[k]["death_v"] == r[0]
            assert recs[k]["birth"].tobytes() == f[u].tobytes() and recs[k]["death"].tobytes() == f[r[0]].tobytes()
        checked[lab] = checked.get(lab, 0) + 1
    log(f"all {picks.size} stratified samples checked against O4: {checked}")


@pytest.mark.parametrize("cfg,scale", [("c1", None), ("c4", 64), ("c5", 96), ("c3", 48), ("c2", 512)])
def test_join_and_split_from_one_read(cfg, scale):
    """f1: mt_compute_join_split reads f once (one tile pass, two tile stores) and gives the merge
    tree of f and the split tree (merge tree of -f, ids still ascending: reading R16) -- each
    bit-exact against O1 with and without the split flag, diagrams included."""
    f, dims, conn = fields.make(cfg, scale=scale)
    a = _lib.MergeTree(dims, conn, device=0)
    b = _lib.MergeTree(dims, conn, device=0)
    tj, ts = _lib.join_split(a, b, torch.from_numpy(f).cuda())
    for mt, T, split in ((a, tj, False), (b, ts, True)):
        rec, npairs, ness = mt.diagram()
        To, po, npo, neo = oracle.merge_tree(f, dims, conn=conn, split=split)
        assert np.array_equal(T.cpu().numpy().view(np.uint64), To), split
        assert (npairs, ness) == (npo, neo)
        assert _lib.pairs_to_numpy(rec).tobytes() == po.tobytes()
