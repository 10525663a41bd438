"""O3 -- the paper's Algorithms 1-5 executed serially (TEST INFRASTRUCTURE).

Follows PAPER.md:242-338 step by step, in the paper's notation, with the
comparisons lifted to (value, id) keys (reading R1) and the two root guards
of reading R4/R5:

- R4: Alg. 3 lines 2-8 climb past T[u] / T[v] only if the cell is not a root
  (a root T[x] = (x, x) has no further pointer; Alg. 4's ``s != v`` guard).
- R5: after a successful CAS (Alg. 3 line 14) the displaced pair is merged
  again (line 15) only if it was not a root.
- R20: Alg. 4 returns the vertex the walk stopped at (``u``), not the printed
  ``v``: when the loop exits on f(s) > a, ``v`` lies below level a in another
  component (counterexample: the "W" path f = [0,4,1,3,2], u = 3).

Serially every CAS succeeds, so Alg. 2 reduces to an assignment.  The edge
order is a parameter: the final (post-repair) store must not depend on it
(SPEC.md "edge-order independence").  Used to check the
readings against O1, never as a reference for the GPU path.
"""
from __future__ import annotations

import numpy as np

from .brute import grid_neighbours, keys


def grid_edges(dims):
    n = dims[0] * dims[1] * dims[2]
    for u in range(n):
        for w in grid_neighbours(u, dims):
            if w > u:
                yield (u, w)


def compute_merge_tree(f, dims, split=False, edge_order=None, seed=None, init=None):
    """``edge_order`` may give any edge list (an explicit graph: dims = (n, 1, 1))."""
    """Alg. 1.  ``init`` optionally replaces line 2-3's (u, u) start state by
    any normalized triplet store of a subgraph (e.g. steepest descent)."""
    dims = tuple(int(d) for d in dims)
    n = dims[0] * dims[1] * dims[2]
    K = keys(f, split)
    T = [(u, u) for u in range(n)] if init is None else [tuple(c) for c in init]   # Alg. 1 l.2-3
    edges = list(grid_edges(dims)) if edge_order is None else list(edge_order)
    if seed is not None:
        rng = np.random.default_rng(seed)
        rng.shuffle(edges)

    def merge(u, s, v):                                   # Alg. 3, iterative
        while True:
            su, up = T[u]
            if up != u and K[su] < K[s]:                  # l.2-4 (+ guard R4)
                u = up
                continue
            sv, vp = T[v]
            if vp != v and K[sv] < K[s]:                  # l.5-8 (+ guard R4)
                v = vp
                continue
            if u == v:                                    # l.9-10
                return
            if K[v] < K[u]:                               # l.11-12
                u, su, up, v, sv, vp = v, sv, vp, u, su, up
            T[v] = (s, u)                                 # l.14, CAS succeeds serially
            if vp == v:                                   # guard R5: displaced a root
                return
            s, v = sv, vp                                 # l.15 Merge(T, u, s_v, v')

    for (a, b) in edges:                                  # Alg. 1 l.4-8
        if K[b] < K[a]:
            merge(a, a, b)
        else:
            merge(b, b, a)

    def representative(u, a):                             # Alg. 4
        s, v = T[u]
        while K[s] <= a and s != v:
            u = v
            s, v = T[u]
        return u       # reading R20: printed "return v" (l.7) is the next, too-deep vertex

    for u in range(n):                                    # Alg. 1 l.9-11, Alg. 5
        s, v = T[u]
        vp = representative(u, K[s])
        if u != vp:
            T[u] = (s, vp)
    return [(u, s, v) for u, (s, v) in enumerate(T)]


def steepest_descent_init(f, dims, split=False):
    """T0[u] = (u, argmin_key lower neighbour) or (u, u): a normalized triplet
    store of the descent forest (derivation B)."""
    dims = tuple(int(d) for d in dims)
    n = dims[0] * dims[1] * dims[2]
    K = keys(f, split)
    T0 = []
    for u in range(n):
        best = u
        for w in grid_neighbours(u, dims):
            if K[w] < K[best]:
                best = w
        T0.append((u, best))
    return T0
