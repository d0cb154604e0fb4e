"""GPU neighbour list is bit-exact with the reference ("neighbor lists bit-exact").

Mirrors test_geom_neighbor.cpp:134-220: multi-image search, cell path vs brute path, FCC blocks,
symmetry; plus the reference-sized C1/C2 lists.
"""
import numpy as np
import pytest

import oracle_lib as O
import paper_2201_01446_b200 as dp

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pot():
    m = dp.make_test_model(3, 2, 2, 4, 1, [64, 64, 64], 6.0, 5.0, 1)
    return dp.DeepPot(m, dp.build_tables(m, 0.1))


def gpu_list(pot, cfg, cutoff):
    c = dp.AtomicConfig(cfg.pos, np.minimum(cfg.type, 2), cfg.h, cfg.periodic)
    return pot.neighbor_list(c, cutoff)


@pytest.mark.parametrize("cutoff", [8.0, 10.0])
def test_c1_lists_bit_exact(pot, cutoff):
    c = dp.gen_config("copper-like", 8, 8, 8, 0.1, 11)
    assert O.lists_equal(gpu_list(pot, c, cutoff), O.or_neighbor_list(c, cutoff))


def test_c2_list_bit_exact(pot):
    c = dp.gen_config("copper-like", 20, 20, 20, 0.1, 11)
    g = gpu_list(pot, c, 10.0)
    o = O.or_neighbor_list(c, 10.0)
    assert g.j.size == o.j.size == 11328898  # SURVEY.md §8 conventions
    assert O.lists_equal(g, o)


@pytest.mark.parametrize("seed", [42, 43, 44])
def test_multi_image_small_box(pot, seed):
    c = dp.make_random_config(12, 2, 6.0, 1.0, seed)  # box edge 6, cutoff 7
    assert O.lists_equal(gpu_list(pot, c, 7.0), O.or_neighbor_list(c, 7.0))


def test_fcc_3x3x3_multi_image(pot):
    c = dp.gen_config("copper-like", 3, 3, 3, 0.0, 1)
    g = gpu_list(pot, c, 8.0)
    assert O.lists_equal(g, O.or_neighbor_list(c, 8.0))
    lens = np.diff(g.offsets)
    assert np.all(lens == lens[0]) and lens[0] > 100


@pytest.mark.parametrize("seed", [7, 8])
def test_cell_path_random(pot, seed):
    c = dp.make_random_config(120, 2, 30.0, 1.2, seed)
    assert O.lists_equal(gpu_list(pot, c, 5.0), O.or_neighbor_list(c, 5.0))


def test_open_and_mixed_boundaries(pot):
    c = dp.make_random_config(40, 2, 12.0, 1.2, 99)
    for per in ([0, 0, 0], [1, 0, 1], [0, 1, 0]):
        cc = dp.AtomicConfig(c.pos, c.type, c.h, per)
        assert O.lists_equal(gpu_list(pot, cc, 6.0), O.or_neighbor_list(cc, 6.0)), per


def test_unwrapped_positions_and_triclinic(pot):
    c = dp.make_random_config(60, 2, 14.0, 1.3, 5)
    rng = np.random.default_rng(0)
    pos = c.pos + 14.0 * rng.integers(-3, 4, size=c.pos.shape)  # atoms far outside the box
    h = np.array([14.0, 0, 0, 2.0, 13.0, 0, -1.5, 1.0, 15.0])
    cc = dp.AtomicConfig(pos, c.type, h)
    assert O.lists_equal(gpu_list(pot, cc, 4.5), O.or_neighbor_list(cc, 4.5))


def test_symmetry(pot):
    c = dp.make_random_config(30, 2, 9.0, 1.2, 3)
    L = gpu_list(pot, c, 6.0)
    ent = set()
    for i in range(c.n_atoms):
        js, ss = L.row(i)
        for j, s in zip(js, ss):
            ent.add((i, int(j), tuple(int(x) for x in s)))
    for (i, j, s) in ent:
        assert (j, i, tuple(-x for x in s)) in ent
