"""O2 -- brute-force definitional checker (TEST INFRASTRUCTURE, tiny inputs).

Reads the triplet definition literally (Sec. 2.1 "Triplet
merge trees"): the triplet of u is (u, s, v) with f(v) < f(u) <= f(s), u and v
in one component of the sublevel set G_{f(s)} = {x : f(x) <= f(s)}
(PAPER.md:130-131), s the first level at which u's branch meets a deeper
vertex, and v the deepest vertex of that component ("minimality",
PAPER.md:198-199, reading R12).  A vertex that is the minimum of its whole
connected component gets (u, u, u).

Ties in f are broken by vertex id (reading R1): keys are (g(x), x) with
g = f, or g = -f for the split tree (reading R16).  Components are found by
breadth-first search on the grid graph (reading R9/R10).  O(n^2) -- n of a few
hundred at most.

The persistence pairs follow from the definition of a branch (PAPER.md:18-22,
180-184): the branch born at minimum u ends at saddle s when u's component
first meets a deeper vertex; a minimum that never does is essential.
"""
from __future__ import annotations

from collections import deque

import numpy as np


def grid_neighbours(u: int, dims):
    nx, ny, nz = dims
    x, y, z = u % nx, (u // nx) % ny, u // (nx * ny)
    if x > 0:
        yield u - 1
    if x + 1 < nx:
        yield u + 1
    if y > 0:
        yield u - nx
    if y + 1 < ny:
        yield u + nx
    if z > 0:
        yield u - nx * ny
    if z + 1 < nz:
        yield u + nx * ny


def keys(f, split=False):
    g = [(-float(x) if split else float(x)) for x in np.asarray(f, dtype=np.float32).reshape(-1)]
    # -0.0 and +0.0 compare equal as floats; tuples compare g first, then id (R1, R2)
    return [(g[i] + 0.0, i) for i in range(len(g))]


def _components(member, dims, adj=None):
    """Label connected components of the vertex set ``member`` by BFS (grid, or adjacency lists)."""
    n = len(member)
    nbrs = (lambda x: adj[x]) if adj is not None else (lambda x: grid_neighbours(x, dims))
    label = [-1] * n
    comps = []
    for s in range(n):
        if not member[s] or label[s] >= 0:
            continue
        cid = len(comps)
        label[s] = cid
        q = deque([s])
        comp = [s]
        while q:
            x = q.popleft()
            for y in nbrs(x):
                if member[y] and label[y] < 0:
                    label[y] = cid
                    q.append(y)
                    comp.append(y)
        comps.append(comp)
    return label, comps


def merge_tree(f, dims, split=False, adj=None):
    """Return (T as list of (u, s, v), finite pairs [(birth_v, death_v)], essential [u]).
    ``adj`` (lists of neighbours) replaces the grid for an explicit graph (dims = (n, 1, 1))."""
    dims = tuple(int(d) for d in dims)
    n = dims[0] * dims[1] * dims[2]
    K = keys(f, split)
    order = sorted(range(n), key=lambda i: K[i])
    trip = [None] * n
    member = [False] * n
    for k, w in enumerate(order):
        # level = key(w): sublevel set {x : key(x) <= key(w)}
        member[w] = True
        label, comps = _components(member, dims, adj)
        cmin = [min(c, key=lambda x: K[x]) for c in comps]
        for u in order[: k + 1]:
            if trip[u] is not None:
                continue
            m = cmin[label[u]]
            if K[m] < K[u]:
                trip[u] = (u, w, m)
    # never met a deeper vertex: minimum of its connected component
    for u in range(n):
        if trip[u] is None:
            trip[u] = (u, u, u)
    finite = [(u, s) for (u, s, v) in trip if s != u]
    ess = [u for (u, s, v) in trip if s == u and v == u]
    return trip, finite, ess


def sublevel_betti0(f, dims, t, split=False):
    """Number of components of {x : g(x) <= t} (by BFS)."""
    g = -np.asarray(f, dtype=np.float32).reshape(-1) if split else np.asarray(f, dtype=np.float32).reshape(-1)
    member = [bool(x <= t) for x in g]
    _, comps = _components(member, tuple(int(d) for d in dims))
    return len(comps)
