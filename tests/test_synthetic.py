"""The product's synthetic-state generator equals the oracle's SplitMix64 fill, and tiles
of a decomposition carry exactly the global field's values."""
import numpy as np

import oracle
from cases import DYCORE_FILLS, DYCORE_SCALARS
from paper_1710_08616_b200 import synthetic


def test_matches_oracle_fill():
    for seed, off, scale in [(0, 0.0, 1.0), (8, 300.0, 1.0), (12, -0.005, 0.01)]:
        a = synthetic.field((7, 13, 5), seed, off, scale)
        b = oracle.fill((7, 13, 5), seed, off, scale)
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_tiles_are_slices_of_the_global_field():
    g = synthetic.field((6, 20, 9), 9, -0.01, 0.02)
    t = synthetic.field((6, 20, 9), 9, -0.01, 0.02, box=[(0, 6), (5, 12), (3, 9)])
    assert np.array_equal(t, g[:, 5:12, 3:9])


def test_dycore_constants_shared():
    assert synthetic.DYCORE_FILLS == DYCORE_FILLS
    assert synthetic.DYCORE_SCALARS == DYCORE_SCALARS
