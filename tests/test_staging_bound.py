"""Derivation N: the diagram records the repair stages per brick are strict
local minima (branch births and roots), an independent set of the grid graph, so a 32 x 16 x 4
brick holds at most 1024 of them and a row of 32 x-consecutive vertices at most 16 -- the fixed
staging runs of the repair rely on it.  Checked with the oracle's diagram, including the
checkerboard that reaches the bound.  CPU only."""
import numpy as np
import pytest

import oracle


def births(f, dims, conn, split=False):
    _, pairs, npairs, ness = oracle.merge_tree(f, dims, conn, split=split)
    return np.asarray(pairs["birth_v"][: npairs + ness], dtype=np.int64)


def per_brick_and_row(b, dims):
    nx, ny, nz = dims
    x, y, z = b % nx, (b // nx) % ny, b // (nx * ny)
    brick = (x // 32) + (nx // 32 + 1) * ((y // 16) + (ny // 16 + 1) * (z // 4))
    row = (x // 32) + (nx // 32 + 1) * (y + ny * z)
    return np.bincount(brick).max(initial=0), np.bincount(row).max(initial=0)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_white_noise_and_ties(seed):
    rng = np.random.default_rng(seed)
    dims = (64, 32, 8)
    for f in (rng.random(int(np.prod(dims))).astype(np.float32),
              rng.integers(0, 3, size=int(np.prod(dims))).astype(np.float32)):
        for split in (False, True):
            mb, mr = per_brick_and_row(births(f, dims, 6, split), dims)
            assert mb <= 1024 and mr <= 16


def test_checkerboard_reaches_the_bound():
    dims = (32, 16, 4)
    x, y, z = np.meshgrid(np.arange(32), np.arange(16), np.arange(4), indexing="ij")
    f = (((x + y + z) % 2).astype(np.float32)).transpose(2, 1, 0).reshape(-1)   # x fastest
    b = births(f, dims, 6)
    mb, mr = per_brick_and_row(b, dims)
    assert mb == 1024 and mr == 16
