"""The paper-method CPU baseline (baseline/paper_cpu: Alg. 1-5 with 64-bit CAS on all host cores,
PAPER.md:242-338) must reach the oracle's store exactly: the post-repair store is unique whatever
the interleaving of the concurrent merges.  CPU only."""
import numpy as np
import pytest

import oracle
from baseline import paper_cpu
from paper_2301_10838_b200 import fields


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_c1_white_noise(seed):
    f, dims, conn = fields.make("c1", seed=seed)
    for split in (False, True):
        T = paper_cpu.merge_tree(f, dims, conn, split=split, threads=4)
        assert np.array_equal(T, oracle.merge_tree(f, dims, conn, split=split)[0])


def test_tie_heavy_grids_both_trees():
    rng = np.random.default_rng(11)
    for _ in range(25):
        d = (int(rng.integers(1, 24)), int(rng.integers(1, 24)), int(rng.integers(1, 12)))
        f = rng.integers(-2, 3, size=d[0] * d[1] * d[2]).astype(np.float32)
        f[rng.random(f.size) < 0.1] = -0.0      # reading R2: -0 and +0 are one value
        conn = 6 if d[2] > 1 else 4
        for split in (False, True):
            T = paper_cpu.merge_tree(f, d, conn, split=split, threads=8)
            assert np.array_equal(T, oracle.merge_tree(f, d, conn, split=split)[0]), (d, split)


def test_larger_fields_all_threads():
    rng = np.random.default_rng(5)
    for d in [(96, 80, 64), (512, 384, 1)]:
        f = rng.random(d[0] * d[1] * d[2]).astype(np.float32)
        conn = 6 if d[2] > 1 else 4
        T = paper_cpu.merge_tree(f, d, conn)
        assert np.array_equal(T, oracle.merge_tree(f, d, conn)[0]), d


def test_rejects_nonfinite_and_bad_args():
    f = np.zeros(8, np.float32)
    f[3] = np.nan
    with pytest.raises(RuntimeError):
        paper_cpu.merge_tree(f, (2, 2, 2), 6)
    with pytest.raises(RuntimeError):
        paper_cpu.merge_tree(np.zeros(8, np.float32), (2, 2, 2), 4)   # 4-conn needs nz == 1
