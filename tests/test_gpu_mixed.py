"""Mixed-precision mode (tcgen05 3xTF32 fitting net + tanh table) against the FP64 oracle.

SURVEY.md §8d / north_star: E, F, virial and E_i within 1e-5 of the FP64 reference on every
preset. The unnormalised descriptor makes the first fitting layer a cancelling sum
(|z| ~ sum|D W| / 45); the forward layers therefore accumulate K in FP64 over short tensor-core
chains (fitting_tc.cu k_tc_fwd64), which keeps even the water preset (E ~ -1.08 eV from 768 atoms
whose E_i cancel) at ~5e-6.
"""
import numpy as np
import pytest

import oracle_lib as O
import paper_2201_01446_b200 as dp

pytestmark = pytest.mark.gpu
TOL = 1e-5


def metrics(r, ro):
    return {"E": abs(r.energy - ro.energy) / abs(ro.energy), "F": O.normwise(r.forces, ro.forces),
            "V": O.normwise(r.virial, ro.virial), "Ei": O.normwise(r.per_atom_energy, ro.per_atom_energy)}


def check(r, ro, tol=None):
    tol = tol or {}
    m = metrics(r, ro)
    print(m)
    for k, v in m.items():
        assert v <= tol.get(k, TOL), (k, v, m)


def test_mixed_c1():
    m = dp.gen_model("copper-like", 7)
    t = dp.build_tables(m, 0.01)
    c = dp.gen_config("copper-like", 8, 8, 8, 0.1, 11)
    ro, co = O.or_compute(c, m, t)
    pot = dp.DeepPot(m, t, precision="mixed")
    r = pot.compute(c)
    check(r, ro)
    assert pot.counters == co


@pytest.mark.parametrize("seed", [500, 501])
def test_mixed_two_types(seed):
    m = dp.make_test_model(2, 6, 8, 20, 2, [18, 18], 6.0, 5.0, 401)
    t = dp.build_tables(m, 0.05)
    c = dp.make_random_config(10, 2, 9.0, 1.8, seed)
    ro, _ = O.or_compute(c, m, t)
    check(dp.DeepPot(m, t, precision="mixed").compute(c), ro)


def test_mixed_water():
    m = dp.gen_model("water-like", 3)
    t = dp.build_tables(m, 0.01)
    c = dp.gen_config("water-like", 4, 4, 4, 0.1, 4)
    ro, _ = O.or_compute(c, m, t)
    check(dp.DeepPot(m, t, precision="mixed").compute(c), ro)


def test_mixed_md_thermo():
    m = dp.gen_model("copper-like", 7)
    t = dp.build_tables(m, 0.01)
    c = dp.gen_config("copper-like", 3, 3, 3, 0.1, 11)
    v = dp.init_velocities(c, m, 330.0, 99)
    mc = dp.MDConfig(n_steps=20, dt=1.0, buffer=2.0, rebuild_every=10, thermo_every=5)
    a = dp.DeepPot(m, t, precision="mixed").run_md(c.copy(), v.copy(), mc)
    b = O.or_run_md(c.copy(), v.copy(), m, t, mc)
    for x, y in zip(a.thermo, b.thermo):
        assert abs(x.pe - y.pe) <= TOL * abs(y.pe)
        # KE after up to 20 steps: per-evaluation force errors (~3e-6) grow along the trajectory
        assert abs(x.ke - y.ke) <= 1e-4 * abs(y.ke)
