"""The counter-based generator (oracle/rng.py) that regenerates shards of the synthetic inputs."""

import numpy as np

from oracle.rng import uniform_block


def test_range_and_determinism():
    a = uniform_block(range(1000), range(8), 2024)
    assert a.shape == (1000, 8) and a.flags.f_contiguous
    assert np.all(a >= 0) and np.all(a < 1)
    assert np.array_equal(a, uniform_block(range(1000), range(8), 2024))
    assert not np.array_equal(a, uniform_block(range(1000), range(8), 2025))
    assert 0.45 < a.mean() < 0.55


def test_slab_is_restriction():
    full = uniform_block(range(200), range(10), 5)
    assert np.array_equal(full[50:80, 3:7], uniform_block(range(50, 80), range(3, 7), 5))


def test_known_values():
    # splitmix64 reference values (seed 0, position (0,0) -> splitmix64(0))
    x = uniform_block([0], [0], 0)[0, 0]
    assert x == (0xE220A8397B1DCDAF >> 11) * 2.0 ** -53


def test_float32_is_cast_of_float64():
    d = uniform_block(range(100), range(3), 9)
    f = uniform_block(range(100), range(3), 9, np.float32)
    assert np.array_equal(d.astype(np.float32), f)
