"""GPU exact (untabulated) path, GPU table build and rmse tooling.

Checked against the compiled reference (oracle/_ref): compute_energy_forces_virial
(exact.cpp:155-173), build_tables (table.cpp:77-162) and rmse_sweep / loglog_slope
(rmse.cpp:63-116). Mirrors test_env_exact.cpp and the accuracy sweep of acceptance.cpp.
"""
import numpy as np
import pytest

import oracle_lib as O
import paper_2201_01446_b200 as dp

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref (compiled reference) not built")]
TOL = 1e-10


def rel(a, b):
    return abs(a - b) / max(abs(a), abs(b), 1e-12)


def check(r, ro, tol=TOL):
    assert rel(r.energy, ro.energy) <= tol, (r.energy, ro.energy)
    assert O.normwise(r.forces, ro.forces) <= tol
    assert O.normwise(r.virial, ro.virial) <= tol
    assert O.normwise(r.per_atom_energy, ro.per_atom_energy) <= tol


@pytest.fixture(scope="module")
def cu():
    return dp.gen_model("copper-like", 7)


def test_exact_c1_copper(cu):
    c = dp.gen_config("copper-like", 8, 8, 8, 0.1, 11)
    check(dp.compute_energy_forces_virial(c, cu), O.ref_compute_exact(c, cu))


@pytest.mark.parametrize("d1,seed", [(6, 501), (8, 502), (20, 503)])
def test_exact_two_types(d1, seed):
    # widths 4*d1 = 24, 32, 80: one, one and three feature registers per lane
    m = dp.make_test_model(2, d1, 4, 20, 2, [40, 40], 6.0, 5.0, seed)
    c = dp.make_random_config(60, 2, 11.0, 1.6, seed)
    check(dp.compute_energy_forces_virial(c, m), O.ref_compute_exact(c, m))


def test_exact_overflow_and_overlap_raise():
    tight = dp.make_test_model(1, 4, 4, 12, 1, [4], 6.0, 5.0, 511)
    c = dp.make_random_config(30, 1, 8.0, 1.5, 5)
    with pytest.raises(dp.NumericalError):
        dp.compute_energy_forces_virial(c, tight)
    m = dp.make_test_model(1, 4, 4, 12, 1, [64], 6.0, 5.0, 512)
    c = dp.make_random_config(10, 1, 9.0, 1.8, 6)
    c.pos[1] = c.pos[0]
    with pytest.raises(dp.NumericalError):
        dp.compute_energy_forces_virial(c, m)


def test_exact_close_to_tabulated(cu):
    # the table at h = 0.001 reproduces the net to O(h^6); E agrees to ~1e-9 relative
    c = dp.gen_config("copper-like", 5, 5, 5, 0.1, 4)
    ex = dp.compute_energy_forces_virial(c, cu)
    tb = dp.compute_energy_forces_virial_tabulated(c, cu, dp.build_tables(cu, 0.001))
    assert rel(ex.energy, tb.energy) < 1e-8
    assert O.normwise(ex.forces, tb.forces) < 1e-5


@pytest.mark.parametrize("h", [0.01, 0.001])
def test_gpu_tables_match_reference(cu, h):
    tg = dp.build_tables_gpu(cu, h)
    tr = O.ref_build_tables(cu, h)
    assert (tg.n, tg.m, tg.block, tg.x0) == (tr.n, tr.m, tr.block, tr.x0)
    assert tg.h == tr.h
    # node values and first derivatives are the net's (tanh ulps apart); a3..a5 are built from
    # differences of O(h^3) and agree to a correspondingly looser relative bound
    stride = tr.interval_stride()
    g = tg.coeffs.reshape(len(tg), tg.n, tg.n_blocks(), 6, tg.block)
    r = tr.coeffs.reshape(len(tr), tr.n, tr.n_blocks(), 6, tr.block)
    assert g.shape[2] * 96 == stride
    np.testing.assert_allclose(g[..., 0:2, :], r[..., 0:2, :], rtol=1e-12, atol=1e-13)
    # evaluated through the tabulated path the two tables give the same physics
    c = dp.gen_config("copper-like", 6, 6, 6, 0.1, 8)
    a = dp.compute_energy_forces_virial_tabulated(c, cu, tg)
    b = dp.compute_energy_forces_virial_tabulated(c, cu, tr)
    check(a, b, 1e-11)


def test_tables_built_on_device_and_installed(cu):
    pot = dp.DeepPot(cu, None)
    c = dp.gen_config("copper-like", 4, 4, 4, 0.1, 9)
    with pytest.raises(dp.InputError):
        pot.compute(c)
    pot.build_tables_gpu(0.01, install=True)
    ref = dp.DeepPot(cu, dp.build_tables(cu, 0.01)).compute(c)
    check(pot.compute(c), ref, 1e-11)


def test_table_build_rejects_bad_step(cu):
    with pytest.raises(dp.InputError):
        dp.build_tables_gpu(cu, 0.0)


def test_rmse_sweep_matches_reference(cu):
    cfgs = [dp.gen_config("copper-like", 4, 4, 4, 0.1, s) for s in (21, 22)]
    hl = [0.04, 0.02, 0.01]
    rows = dp.rmse_sweep(cu, hl, cfgs)
    re, rf, slope = O.ref_rmse_sweep(cu, hl, cfgs)
    for row, e, f in zip(rows, re, rf):
        assert rel(row.rmse_e, e) < 1e-5, (row.rmse_e, e)
        assert rel(row.rmse_f, f) < 1e-5, (row.rmse_f, f)
    s = dp.loglog_slope(rows)
    assert abs(s - slope) < 1e-3
    assert s > 4.0  # quintic Hermite: O(h^6) energy error


def test_rmse_compare_zero_for_identical_paths(cu):
    c = dp.gen_config("copper-like", 4, 4, 4, 0.1, 23)
    rep = dp.rmse_compare(cu, dp.build_tables(cu, 0.001), [c])
    assert rep.n_configs == 1
    assert 0.0 < rep.rmse_e < 1e-8 and 0.0 < rep.rmse_f < 1e-5
