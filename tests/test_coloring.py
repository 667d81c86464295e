"""Host coloring (paper_2507_11512_b200/coloring.py) against the reference:
greedy closed form and the vectorised JPL (ref: coloring.py:36-123,
tests/test_coloring.py)."""
import numpy as np
import pytest

from conftest import load_golden
from paper_2507_11512_b200.coloring import _local_neighbours, color, greedy_coloring, jpl_coloring


@pytest.mark.parametrize("key", ["4x4x4_s0", "6x4x8_s3", "8x8x8_s11", "5x3x4_s7", "16x16x16_s0"])
def test_jpl_bitwise_vs_reference(key):
    g = load_golden("jpl.npz")
    dims, seed = key.split("_s")
    lx, ly, lz = map(int, dims.split("x"))
    c = jpl_coloring(lx, ly, lz, int(seed))
    np.testing.assert_array_equal(c.color, g["color_" + key])
    np.testing.assert_array_equal(c.perm, g["perm_" + key])
    np.testing.assert_array_equal(c.color_offsets, g["offsets_" + key])


def _valid(lx, ly, lz, col):
    n = lx * ly * lz
    nb = _local_neighbours(lx, ly, lz, np.arange(n))
    cn = np.where(nb >= 0, col.color[np.where(nb >= 0, nb, 0)], -1)
    return not np.any(cn == col.color[:, None])


def test_jpl_valid_for_many_seeds():
    # ref: tests/test_coloring.py:42-47 (100 seeds, 4^3); here 40 seeds on 6x5x4
    for seed in range(40):
        c = jpl_coloring(6, 5, 4, seed)
        assert _valid(6, 5, 4, c)
        assert c.num_colors <= 27


def test_jpl_deterministic_per_seed():
    a, b = jpl_coloring(8, 8, 8, 11), jpl_coloring(8, 8, 8, 11)
    assert np.array_equal(a.color, b.color)


def test_greedy_counts():
    # ref: tests/test_acceptance.py:227-242 -> 8 colors in 3D
    c = greedy_coloring(8, 8, 8)
    assert c.num_colors == 8 and _valid(8, 8, 8, c)
    assert color((4, 4, 4)).num_colors == 8


def test_unknown_strategy():
    with pytest.raises(ValueError):
        color((4, 4, 4), "bogus")
