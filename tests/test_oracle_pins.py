"""Pins of the oracle O1 against things other than itself (CPU only).

- golden fixtures worked by hand from the paper's definitions (tests/golden/*.txt, cited inside);
- O2, the definition read literally (BFS over sublevel sets), exhaustively on all value orders
  of tiny grids and on random tie-heavy tiny grids;
- O3, the paper's Algorithms 1-5 run serially in random edge orders (checks readings R4/R5/R20);
- closed-form families (constant, ramps, checkerboards);
- a library routine: scipy.ndimage.label component counts of sublevel sets vs the diagram;
- structural invariants I1-I4 at moderate sizes.
"""
import itertools

import numpy as np
import pytest
from scipy import ndimage

import oracle
from oracle import alg1, brute, invariants
from paper_2301_10838_b200 import fields
from golden_io import all_cases

GOLDEN = all_cases()


def o1_triplets(f, dims, conn, split=False):
    T, pairs, npairs, ness = oracle.merge_tree(f, dims, conn=conn, split=split)
    s, v = oracle.unpack(T)
    return [(u, int(s[u]), int(v[u])) for u in range(T.size)], pairs, npairs, ness


@pytest.mark.parametrize("case", GOLDEN, ids=[c["name"] for c in GOLDEN])
def test_golden(case):
    trip, pairs, npairs, ness = o1_triplets(case["f"], case["dims"], case["conn"], case["split"])
    assert trip == case["triplets"]
    fin = [(int(p["birth_v"]), int(p["death_v"])) for p in pairs[:npairs]]
    assert fin == case["pairs"]
    ess = [int(p["birth_v"]) for p in pairs[npairs:]]
    assert ess == case["essential"]
    f = case["f"]
    for p in pairs[:npairs]:  # values copied bit-exact from the input f (reading R14)
        assert p["birth"].tobytes() == f[p["birth_v"]].tobytes()
        assert p["death"].tobytes() == f[p["death_v"]].tobytes()
    for p in pairs[npairs:]:
        assert p["death_v"] == p["birth_v"] and np.isinf(p["death"]) and p["death"] > 0


@pytest.mark.parametrize("dims,conn", [((3, 2, 1), 4), ((6, 1, 1), 4), ((1, 2, 3), 6)])
def test_o1_equals_definition_all_orders(dims, conn):
    """All 720 value orders of a 6-vertex grid: O1 == O2 (definition by BFS)."""
    for perm in itertools.permutations(range(6)):
        f = np.array(perm, dtype=np.float32)
        trip, _, npairs, ness = o1_triplets(f, dims, conn)
        b_trip, b_fin, b_ess = brute.merge_tree(f, dims)
        assert trip == b_trip, (perm, trip, b_trip)
        assert npairs == len(b_fin) and ness == len(b_ess)


def test_o1_equals_definition_random_tiny():
    rng = np.random.default_rng(12345)
    for it in range(250):
        dims = tuple(int(x) for x in rng.integers(1, 6, 3))
        n = int(np.prod(dims))
        if it % 3 == 0:
            f = rng.integers(0, 3, n).astype(np.float32)          # heavy ties
        elif it % 3 == 1:
            f = rng.standard_normal(n).astype(np.float32)
        else:
            f = (rng.integers(-2, 3, n) * 0.0).astype(np.float32)  # +-0.0 mix
            f[rng.random(n) < 0.5] *= -1
        split = bool(it % 2)
        trip, pairs, npairs, ness = o1_triplets(f, dims, 6, split)
        b_trip, b_fin, b_ess = brute.merge_tree(f, dims, split)
        assert trip == b_trip
        assert [(int(p["birth_v"]), int(p["death_v"])) for p in pairs[:npairs]] == sorted(b_fin)
        assert [int(p["birth_v"]) for p in pairs[npairs:]] == b_ess


def test_o1_equals_paper_algorithm_any_edge_order():
    """O3 (Alg. 1-5 serially, random edge orders, both start states) == O1."""
    rng = np.random.default_rng(7)
    for it in range(120):
        dims = tuple(int(x) for x in rng.integers(1, 7, 3))
        n = int(np.prod(dims))
        f = (rng.integers(0, 5, n) if it % 2 else rng.random(n)).astype(np.float32)
        trip, *_ = o1_triplets(f, dims, 6)
        assert alg1.compute_merge_tree(f, dims, seed=it) == trip
        init = alg1.steepest_descent_init(f, dims)
        assert alg1.compute_merge_tree(f, dims, seed=it + 99, init=init) == trip


@pytest.mark.parametrize("dims", [(20, 17, 9), (33, 1, 1), (1, 1, 40), (16, 16, 1)])
def test_closed_form_constant_and_ramps(dims):
    nx, ny, nz = dims
    n = nx * ny * nz
    conn = 4 if nz == 1 else 6
    u = np.arange(n)
    # constant: id order decides, unique minimum 0, every other vertex regular (u, u, 0)
    T, _, npairs, ness = oracle.merge_tree(np.full(n, 2.5, np.float32), dims, conn)
    s, v = oracle.unpack(T)
    assert np.all(s == u) and np.all(v == 0) and npairs == 0 and ness == 1
    # ramp x+y+z: same store
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    ramp = (x + y + z).astype(np.float32).reshape(-1)
    T, _, npairs, ness = oracle.merge_tree(ramp, dims, conn)
    s, v = oracle.unpack(T)
    assert np.all(s == u) and np.all(v == 0) and npairs == 0
    # reversed ramp: unique minimum at the far corner n-1
    T, _, npairs, ness = oracle.merge_tree(-ramp, dims, conn)
    s, v = oracle.unpack(T)
    assert np.all(s == u) and np.all(v == n - 1) and npairs == 0


@pytest.mark.parametrize("dims", [(12, 10, 7), (31, 23, 1), (2, 2, 2)])
def test_closed_form_checkerboard(dims):
    """f = (x+y+z) mod 2: every even vertex is a strict local minimum; all of them but vertex 0
    die at value 1: diagram {(0,1)} x (n_even - 1) + essential (0, inf)."""
    nx, ny, nz = dims
    conn = 4 if nz == 1 else 6
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    f = ((x + y + z) % 2).astype(np.float32).reshape(-1)
    n_even = int((f == 0).sum())
    T, pairs, npairs, ness = oracle.merge_tree(f, dims, conn)
    assert npairs == n_even - 1 and ness == 1
    assert np.all(pairs["birth"][:npairs] == 0) and np.all(pairs["death"][:npairs] == 1)
    assert np.array_equal(np.sort(pairs["birth_v"][:npairs]), np.nonzero(f == 0)[0][1:])
    assert pairs["birth_v"][npairs] == 0
    s, v = oracle.unpack(T)
    assert np.all(f[s[:npairs]] >= 0)
    invariants.check(T, f, dims, n_pairs=npairs, n_ess=ness)


def _beta0_checks(f, dims, conn, split, thresholds):
    T, pairs, npairs, ness = oracle.merge_tree(f, dims, conn=conn, split=split)
    nx, ny, nz = dims
    g = (-f if split else f).reshape(nz, ny, nx)
    if nz == 1:
        g = g[0]
    struct = ndimage.generate_binary_structure(g.ndim, 1)  # 4-/6-connectivity
    b = pairs["birth"].astype(np.float64)
    d = pairs["death"].astype(np.float64)
    if split:  # split tree pairs hold input values; compare in -f
        b, d = -b, np.where(np.isinf(d), np.inf, -d)
    for t in thresholds:
        _, ncomp = ndimage.label(g <= t, structure=struct)
        assert ncomp == int(np.sum((b <= t) & (t < d))), t
    return T, npairs, ness


@pytest.mark.parametrize("cfg,scale,split", [("c1", 24, False), ("c1", 24, True), ("c2", 96, False),
                                             ("c3", 32, False), ("c4", 20, True)])
def test_diagram_betti0_library(cfg, scale, split):
    """Library pin: scipy.ndimage.label counts components of {g <= t}; the diagram must give
    #{birth <= t < death} for every sampled threshold (ties included: the sublevel set at t
    is a prefix of the id-tiebroken order)."""
    f, dims, conn = fields.make(cfg, scale=scale)
    g = -f if split else f
    ts = np.quantile(g, np.linspace(0.0, 1.0, 41))
    ts = np.concatenate([ts, np.unique(g)[:: max(1, g.size // 50)]])
    T, npairs, ness = _beta0_checks(f, dims, conn, split, ts)
    invariants.check(T, f, dims, split=split, n_pairs=npairs, n_ess=ness)


def test_split_is_merge_tree_of_negation():
    rng = np.random.default_rng(3)
    for it in range(30):
        dims = tuple(int(x) for x in rng.integers(1, 9, 3))
        n = int(np.prod(dims))
        f = (rng.integers(0, 6, n) if it % 2 else rng.standard_normal(n)).astype(np.float32)
        Ts, *_ = oracle.merge_tree(f, dims, 6, split=True)
        Tn, *_ = oracle.merge_tree(-f, dims, 6, split=False)
        assert np.array_equal(Ts, Tn)


@pytest.mark.parametrize("cfg,scale", [("c1", None), ("c4", 48), ("c3", 48), ("c2", 256)])
def test_invariants_moderate(cfg, scale):
    f, dims, conn = fields.make(cfg, scale=scale)
    T, pairs, npairs, ness = oracle.merge_tree(f, dims, conn)
    invariants.check(T, f, dims, n_pairs=npairs, n_ess=ness)
    # pairs are the minima (other than the global one), each dying at a higher-or-equal value
    assert np.all(pairs["birth"][:npairs] <= pairs["death"][:npairs])
    assert np.all(np.diff(pairs["birth_v"][:npairs].astype(np.int64)) > 0)


def test_errors_and_empty():
    with pytest.raises(oracle.OracleError) as e:
        oracle.merge_tree(np.array([0, np.nan], np.float32), (2, 1, 1), 4)
    assert e.value.status == oracle.NONFINITE
    with pytest.raises(oracle.OracleError) as e:
        oracle.merge_tree(np.array([0, np.inf], np.float32), (2, 1, 1), 4)
    assert e.value.status == oracle.NONFINITE
    with pytest.raises(oracle.OracleError) as e:
        oracle.merge_tree(np.zeros(8, np.float32), (2, 2, 2), 4)
    assert e.value.status == oracle.INVALID
    T, pairs, npairs, ness = oracle.merge_tree(np.zeros(0, np.float32), (0, 4, 4), 6)
    assert T.size == 0 and npairs == 0 and ness == 0


def test_field_generators_deterministic():
    a = fields.u24(1, 4096)
    b = fields.u24(1, 4096)
    assert np.array_equal(a, b)
    assert np.all((a >= 0) & (a < 1))
    assert np.all(a * 2 ** 24 == np.round(a * 2 ** 24))  # exactly on the 2^-24 grid
    assert fields.field_hash(a) == fields.field_hash(b)


def test_filter_by_persistence_definition():
    """SPEC.md analysis examples: P3 diagram {(2,3)} ess {1}: eps 0.5 keeps the pair, eps 2 drops it,
    eps 0 keeps every positive-persistence pair; essential classes always stay."""
    f = np.array([1, 3, 2], np.float32)
    T, pairs, npairs, ness = oracle.merge_tree(f, (3, 1, 1), 4)
    assert oracle.filter_by_persistence(pairs, npairs, 0.5).tolist() == pairs.tolist()
    kept = oracle.filter_by_persistence(pairs, npairs, 2.0)
    assert kept.size == 1 and kept[0]["birth_v"] == 0 and np.isinf(kept[0]["death"])
    f = np.array([0, 1, 0], np.float32)   # tie pair (0, 1) has persistence 1; zero-persistence pairs drop at eps 0
    T, pairs, npairs, ness = oracle.merge_tree(np.array([1, 1, 0, 1], np.float32), (4, 1, 1), 4)
    assert all(p["death"] - p["birth"] == 0 for p in pairs[:npairs])
    assert oracle.filter_by_persistence(pairs, npairs, 0.0).size == ness


@pytest.mark.parametrize("cfg,scale,split", [("c1", 16, False), ("c4", 20, True), ("c5", 24, False), ("c2", 48, False),
                                             ("c3", 20, True)])
def test_o4_single_vertex_triplets_equal_o1(cfg, scale, split):
    """O4 (bounded floods from one vertex, the definition) against O1 on every
    vertex of small grids of each recipe, both tree directions: O4 is what the full-size GPU test
    samples with."""
    f, dims, conn = fields.make(cfg, scale=scale)
    T, _, _, _ = oracle.merge_tree(f, dims, conn=conn, split=split)
    n = int(np.prod(dims))
    for u in range(n):
        r = oracle.triplet_at(f, dims, conn, u, split=split, cap=n)
        assert r is not None
        assert (np.uint64(r[0]) << np.uint64(32)) | np.uint64(r[1]) == T[u], (u, r, divmod(int(T[u]), 1 << 32))


def test_o4_cap_skips():
    f, dims, conn = fields.make("c1")
    T, _, _, _ = oracle.merge_tree(f, dims, conn=conn)
    root = int(np.flatnonzero((T >> np.uint64(32)) == (T & np.uint64(0xffffffff)))[0])
    assert oracle.triplet_at(f, dims, conn, root, cap=100) is None   # the global minimum floods everything
    assert oracle.triplet_at(f, dims, conn, root, cap=f.size) == (root, root)


def test_o4_ids_past_2_32_hand_derived():
    """O4 with 64-bit ids (PAPER.md:389-396 stops at 32 bits) on a
    2048 x 2048 x 1032 grid (4.33e9 vertices; plane 1024 starts at id 2^32 exactly), f = 0
    except two pits joined by a path along +z that crosses id 2^32 (an anonymous zero mapping:
    only the touched pages exist).  By the definition:
      B = -1 (plane 1022) -> p1 = -0.9 -> p2 = -0.8 (plane 1024, id >= 2^32) -> p3 = -0.7 -> A = -2;
      T[p1] = (p1, B): p1 has a lower neighbour, its component at level f(p1) is {B, p1};
      T[p3] = (p3, A): at level f(p3) the path joins A, the deepest vertex;
      T[B]  = (p3, A): B's component first reaches a deeper vertex (A) at level f(p3);
    truncating any id (or a neighbour offset) to 32 bits breaks one of these."""
    import mmap
    dims = (2048, 2048, 1032)
    nx, ny, nz = dims
    n, sxy = nx * ny * nz, nx * ny
    m = mmap.mmap(-1, n * 4)
    try:
        f = np.frombuffer(m, dtype=np.float32)
        b = 1022 * sxy + 9 * nx + 7
        p1, p2, p3, a = b + sxy, b + 2 * sxy, b + 3 * sxy, b + 4 * sxy
        assert p1 < 2 ** 32 <= p2
        for x, val in ((b, -1.0), (p1, -0.9), (p2, -0.8), (p3, -0.7), (a, -2.0)):
            f[x] = val
        assert oracle.triplet_at(f, dims, 6, p1, cap=64) == (p1, b)
        assert oracle.triplet_at(f, dims, 6, p2, cap=64) == (p2, b)
        assert oracle.triplet_at(f, dims, 6, p3, cap=64) == (p3, a)
        assert oracle.triplet_at(f, dims, 6, b, cap=64) == (p3, a)
        assert oracle.triplet_at(f, dims, 6, a, cap=64) is None          # the global minimum floods all
        # a zero vertex's sublevel component holds every lower-id zero: far past the cap
        assert oracle.triplet_at(f, dims, 6, a + 1, cap=64) is None
        del f
    finally:
        m.close()
