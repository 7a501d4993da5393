"""The device generators (csrc/generate.cu) reproduce generators.py bit-for-bit."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,seed,start,n", [("sphere", 1, 0, 200_000), ("terrain", 2, 12_345, 200_000),
                                              ("scene", 3, 7, 200_000), ("cluster", 4, 0, 600_000),
                                              ("surface", 5, 3, 100_000)])
def test_device_generator_matches_numpy(kind, seed, start, n):
    import torch

    import bench
    from paper_2302_14801_b200.device import unpack_records
    from paper_2302_14801_b200.generators import synthetic_rows
    d = bench.make_input_device(torch, kind, n, seed, start=start)
    pos_d, col_d = unpack_records(d.cpu().numpy(), 0)
    pos_h, col_h = synthetic_rows(kind, seed, start, n)
    assert np.array_equal(pos_d.astype(np.float32), pos_h)
    assert np.array_equal(col_d, col_h)
