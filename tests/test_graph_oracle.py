"""Explicit graphs: pins of the graph oracle on CPU.

SPEC.md examples worked from the paper's definitions: the edgeless graph
(S:250), two components, the star graph; then O1 == O2 (BFS definition over
adjacency lists) and O1 == O3 (the paper's Alg. 1-5 serially) on random graphs with several
components, self-loops and duplicate edges; a grid given as CSR equals the grid oracle."""
import numpy as np
import pytest

import oracle
from oracle import alg1, brute


def trip(T):
    s, v = oracle.unpack(T)
    return [(u, int(s[u]), int(v[u])) for u in range(T.size)]


def test_spec_examples():
    # edgeless graph, n = 4: every vertex is the minimum of its own component
    row, col = oracle.csr_from_edges(4, [])
    T, pairs, npairs, ness = oracle.merge_tree_graph(np.array([5, 1, 2, 0], np.float32), row, col)
    assert trip(T) == [(0, 0, 0), (1, 1, 1), (2, 2, 2), (3, 3, 3)] and npairs == 0 and ness == 4
    assert [int(p["birth_v"]) for p in pairs] == [0, 1, 2, 3]
    # two components: path 0-1 and the isolated vertex 2, f = [0, 1, 5]
    row, col = oracle.csr_from_edges(3, [(0, 1)])
    T, pairs, npairs, ness = oracle.merge_tree_graph(np.array([0, 1, 5], np.float32), row, col)
    assert trip(T) == [(0, 0, 0), (1, 1, 0), (2, 2, 2)] and (npairs, ness) == (0, 2)
    # star graph f = [0, 2, 3], edges (0,1), (0,2)
    row, col = oracle.csr_from_edges(3, [(0, 1), (0, 2)])
    T, pairs, npairs, ness = oracle.merge_tree_graph(np.array([0, 2, 3], np.float32), row, col)
    assert trip(T) == [(0, 0, 0), (1, 1, 0), (2, 2, 0)]
    # the P3 path as a graph
    row, col = oracle.csr_from_edges(3, [(0, 1), (1, 2)])
    T, pairs, npairs, ness = oracle.merge_tree_graph(np.array([1, 3, 2], np.float32), row, col)
    assert trip(T) == [(0, 0, 0), (1, 1, 0), (2, 1, 0)]


def random_graph(rng, n, p, loops=True, dups=True):
    iu = np.triu_indices(n, 1)
    m = rng.random(iu[0].size) < p
    edges = list(zip(iu[0][m].tolist(), iu[1][m].tolist()))
    if loops and n:
        edges += [(int(x), int(x)) for x in rng.integers(0, n, 2)]
    if dups and edges:
        edges += edges[: max(1, len(edges) // 5)]
    return edges


def test_graph_oracle_equals_definition_and_algorithm():
    rng = np.random.default_rng(2301)
    for it in range(150):
        n = int(rng.integers(1, 24))
        edges = random_graph(rng, n, float(rng.choice([0.05, 0.15, 0.4])))
        f = (rng.integers(0, 4, n) if it % 2 else rng.standard_normal(n)).astype(np.float32)
        row, col = oracle.csr_from_edges(n, edges)
        split = bool(it % 3 == 0)
        T, pairs, npairs, ness = oracle.merge_tree_graph(f, row, col, split)
        adj = [col[row[u]:row[u + 1]].tolist() for u in range(n)]
        b_trip, b_fin, b_ess = brute.merge_tree(f, (n, 1, 1), split, adj=adj)
        assert trip(T) == b_trip
        assert [(int(p["birth_v"]), int(p["death_v"])) for p in pairs[:npairs]] == sorted(b_fin)
        assert [int(p["birth_v"]) for p in pairs[npairs:]] == b_ess
        plain = [(a, b) for a, b in edges if a != b]
        assert alg1.compute_merge_tree(f, (n, 1, 1), split, edge_order=plain, seed=it) == b_trip


@pytest.mark.parametrize("dims", [(7, 5, 3), (12, 9, 1)])
def test_grid_as_graph(dims):
    nx, ny, nz = dims
    n = nx * ny * nz
    f = np.random.default_rng(n).integers(0, 6, n).astype(np.float32)
    edges = [(u, w) for u in range(n) for w in brute.grid_neighbours(u, dims) if w > u]
    row, col = oracle.csr_from_edges(n, edges)
    Tg, pg, _, _ = oracle.merge_tree_graph(f, row, col)
    T, p, _, _ = oracle.merge_tree(f, dims, 4 if nz == 1 else 6)
    assert np.array_equal(T, Tg) and p.tobytes() == pg.tobytes()
