"""The bench's input generator equals the oracle's (same seeded arrays)."""

import numpy as np

from oracle.arrayneat_oracle import synthetic_population as oracle_gen
from paper_2404_01817_b200.synthetic import synthetic_population as bench_gen


def test_generators_identical():
    for variant in ("T", "M"):
        a = oracle_gen(5, 128, 512, 32, 8, seed=9, variant=variant)
        b = bench_gen(5, 128, 512, 32, 8, seed=9, variant=variant)
        assert np.array_equal(a[0], b[0], equal_nan=True)
        assert np.array_equal(a[1], b[1], equal_nan=True)
