"""Parity on the configurations bench.py reports, against the LIVE reference (oracle/_ref).

VERDICT r01 "Next #1": the benchmarked systems themselves are compared with the unmodified
reference library, not only the 2,048-atom C1 case:
  * C2 (Cu 20^3 = 32,000 atoms): compute_energy_forces_virial_tabulated (fused.cpp:245-288) with
    every host thread -- E, F, virial, E_i within 1e-10 normwise, FusedCounters equal;
  * C2 10-step NVE run_md (md.cpp:151-231) -- thermo and final state;
  * C3 (Cu 64^3 = 1,048,576 atoms): one evaluation against the reference (slow: ~3 min of CPU);
  * C3 mixed precision against the FP64 path at 1e-5 (north_star's separately reported mode).
Inputs are made by the reference's own generators (gen_model / build_tables / gen_config /
init_velocities through oracle/ref_shim.cpp), so nothing of the product shapes them.
"""
import os

import numpy as np
import pytest

import oracle_lib as O
import paper_2201_01446_b200 as dp

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built")]
TOL = 1e-10
THREADS = os.cpu_count() or 1


def rel(a, b):
    return abs(a - b) / max(abs(a), abs(b), 1e-300)


def check(r, ro, tol=TOL):
    m = {"E": rel(r.energy, ro.energy), "F": O.normwise(r.forces, ro.forces),
         "V": O.normwise(r.virial, ro.virial), "Ei": O.normwise(r.per_atom_energy, ro.per_atom_energy)}
    print(m)
    for k, v in m.items():
        assert v <= tol, (k, v, m)
    return m


@pytest.fixture(scope="module")
def cu():
    m = O.ref_gen_model("copper-like", 7)
    t = O.ref_build_tables(m, 0.01)
    return m, t


def test_c2_eval_vs_reference(cu):
    m, t = cu
    c = O.ref_gen_config("copper-like", 20, 20, 20, 0.1, 11)
    ro, co, _ = O.ref_compute(c, m, t, m.r_cut + 2.0, THREADS)
    # the reference's C2 energy
    assert ro.energy == -5040.6583216965946
    pot = dp.DeepPot(m, t)
    pot.set_skin(2.0)
    r = pot.compute(c)
    check(r, ro)
    assert pot.counters == co
    assert co.rows_forward == co.rows_backward and co.extrapolations == 0
    pot.close()


def test_c2_ten_step_md_vs_reference(cu):
    m, t = cu
    c = O.ref_gen_config("copper-like", 20, 20, 20, 0.1, 11)
    v = O.ref_init_velocities(c, m, 330.0, 99)
    mc = dp.MDConfig(n_steps=10, dt=1.0, buffer=2.0, rebuild_every=50, thermo_every=5)
    ca, va = c.copy(), v.copy()
    cb, vb = c.copy(), v.copy()
    a = dp.DeepPot(m, t).run_md(ca, va, mc)
    b = O.ref_run_md(cb, vb, m, t, mc, THREADS)
    assert a.force_evals == b.force_evals == 11
    assert a.staleness_checks == b.staleness_checks
    assert [x.step for x in a.thermo] == [y.step for y in b.thermo] == [0, 5, 10]
    for x, y in zip(a.thermo, b.thermo):
        assert rel(x.pe, y.pe) <= TOL, (x.pe, y.pe)
        assert rel(x.ke, y.ke) <= TOL, (x.ke, y.ke)
        assert rel(x.pressure, y.pressure) <= 1e-9, (x.pressure, y.pressure)
    assert rel(a.final_total, b.final_total) <= TOL
    assert O.normwise(ca.pos, cb.pos) <= TOL
    assert O.normwise(va, vb) <= 1e-9
    assert a.counters == b.counters


@pytest.mark.slow
@pytest.mark.timeout(2400)
def test_c3_eval_vs_reference(cu):
    m, t = cu
    c = O.ref_gen_config("copper-like", 64, 64, 64, 0.1, 11)
    pot = dp.DeepPot(m, t)
    r = pot.compute(c)
    cnt = pot.counters
    pot.close()
    ro, co, secs = O.ref_compute(c, m, t, 0.0, THREADS)
    print(f"reference C3: list {secs[0]:.1f} s, eval {secs[1]:.1f} s on {THREADS} threads")
    check(r, ro)
    assert cnt == co


@pytest.fixture(scope="module")
def c3_fp64(cu):
    m, t = cu
    c = O.ref_gen_config("copper-like", 64, 64, 64, 0.1, 11)
    pot = dp.DeepPot(m, t)
    r = pot.compute(c)
    pot.close()
    return c, r


@pytest.mark.slow
def test_c3_mixed_vs_fp64(cu, c3_fp64):
    m, t = cu
    c, ro = c3_fp64
    pot = dp.DeepPot(m, t, precision="mixed")
    r = pot.compute(c)
    pot.close()
    check(r, ro, 1e-5)


def test_c2_mixed_vs_reference(cu):
    m, t = cu
    c = O.ref_gen_config("copper-like", 20, 20, 20, 0.1, 11)
    ro, co, _ = O.ref_compute(c, m, t, 0.0, THREADS)
    pot = dp.DeepPot(m, t, precision="mixed")
    check(pot.compute(c), ro, 1e-5)
    assert pot.counters == co
    pot.close()
