"""Structural invariants of a finished triplet store (TEST INFRASTRUCTURE).

I1  non-root cells: key(v) < key(u) <= key(s); root <=> s = v = u
    (f(v) < f(u) <= f(s); (u,u,u) for the component minimum)
I2  non-root cells: s = u  <=>  u has a lower neighbour (regular / saddle
    vertex, "(u, u, v)" PAPER.md:193-195); s != u exactly at local minima
    that are not component minima
I3  #roots = #connected components (one for every non-empty grid)
I4  #finite pairs = #strict local minima - #components
I5  u -> v is a forest: following v strictly decreases the key (implied by I1)
All checks are vectorised numpy so they run at full size.
"""
from __future__ import annotations

import numpy as np


def order_keys(f, split=False):
    """Rank of every vertex in the (g(x), x) total order (reading R1/R2/R16),
    computed with a stable sort on plain float values (library sort)."""
    g = np.asarray(f, dtype=np.float32).reshape(-1).astype(np.float64)
    if split:
        g = -g
    g = g + 0.0  # -0.0 -> +0.0 (they compare equal anyway)
    order = np.argsort(g, kind="stable")  # stable => ties by ascending id
    rank = np.empty(order.size, dtype=np.int64)
    rank[order] = np.arange(order.size, dtype=np.int64)
    return rank


def lower_neighbour_exists(rank, dims):
    nx, ny, nz = dims
    r = rank.reshape(nz, ny, nx)
    has = np.zeros_like(r, dtype=bool)
    has[:, :, 1:] |= r[:, :, :-1] < r[:, :, 1:]
    has[:, :, :-1] |= r[:, :, 1:] < r[:, :, :-1]
    has[:, 1:, :] |= r[:, :-1, :] < r[:, 1:, :]
    has[:, :-1, :] |= r[:, 1:, :] < r[:, :-1, :]
    has[1:, :, :] |= r[:-1, :, :] < r[1:, :, :]
    has[:-1, :, :] |= r[1:, :, :] < r[:-1, :, :]
    return has.reshape(-1)


def check(T, f, dims, split=False, n_pairs=None, n_ess=None):
    """Raise AssertionError on the first violated invariant; return counts."""
    T = np.asarray(T, dtype=np.uint64)
    n = T.size
    u = np.arange(n, dtype=np.int64)
    s = (T >> np.uint64(32)).astype(np.int64)
    v = (T & np.uint64(0xFFFFFFFF)).astype(np.int64)
    assert np.all(s < n) and np.all(v < n), "I0: ids in range"
    rank = order_keys(f, split)
    root = (s == u) & (v == u)
    nonroot = ~root
    assert np.all(rank[v[nonroot]] < rank[u[nonroot]]), "I1: key(v) < key(u)"
    assert np.all(rank[u[nonroot]] <= rank[s[nonroot]]), "I1: key(u) <= key(s)"
    assert not np.any((v == u) & (s != u)), "I1: v = u only at roots"
    lower = lower_neighbour_exists(rank, dims)
    assert np.all((s[nonroot] == u[nonroot]) == lower[nonroot]), "I2: s = u <=> lower neighbour"
    n_roots = int(root.sum())
    if n:
        assert n_roots == 1, "I3: one root per connected grid"
    n_min = int((~lower).sum())
    n_fin = int((nonroot & (s != u)).sum())
    assert n_fin == n_min - n_roots, "I4: #pairs = #minima - #components"
    if n_pairs is not None:
        assert n_pairs == n_fin
    if n_ess is not None:
        assert n_ess == n_roots
    return {"n_roots": n_roots, "n_minima": n_min, "n_pairs": n_fin}


def betti0_from_diagram(pairs, t):
    """#{finite pairs with birth <= t < death} + #{essential with birth <= t}."""
    b = pairs["birth"].astype(np.float64)
    d = pairs["death"].astype(np.float64)
    return int(np.sum((b <= t) & (t < d)))
