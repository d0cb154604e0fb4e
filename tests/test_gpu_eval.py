"""GPU energy/force/virial parity with the CPU oracle (FP64, 1e-10 normwise).

Mirrors the reference's own tests: fused path vs its oracle (test_fused.cpp:23-57), padding
invariance (:77-106), counters (:108-157), FD forces and virial (acceptance.cpp:157-222),
invariances and force balance (:225-308), zero forces on the perfect lattice (test_io.cpp:201-216).
"""
import numpy as np
import pytest

import oracle_lib as O
import paper_2201_01446_b200 as dp

pytestmark = pytest.mark.gpu
TOL = 1e-10


def rel(a, b):
    return abs(a - b) / max(abs(a), abs(b), 1e-12)


def check(r, ro, cnt=None, cnto=None, tol=TOL):
    assert rel(r.energy, ro.energy) <= tol, (r.energy, ro.energy)
    assert O.normwise(r.forces, ro.forces) <= tol
    assert O.normwise(r.virial, ro.virial) <= tol
    assert O.normwise(r.per_atom_energy, ro.per_atom_energy) <= tol
    if cnt is not None:
        assert cnt == cnto


@pytest.fixture(scope="module")
def cu():
    m = dp.gen_model("copper-like", 7)
    t = dp.build_tables(m, 0.01)
    return m, t, dp.DeepPot(m, t)


def test_c1_parity(cu):
    m, t, pot = cu
    c = dp.gen_config("copper-like", 8, 8, 8, 0.1, 11)
    ro, co = O.or_compute(c, m, t)
    r = pot.compute(c)
    check(r, ro, pot.counters, co)
    assert co.rows_forward == co.rows_backward == 363556


def test_c1_fine_table(cu):
    m, _, _ = cu
    t = dp.build_tables(m, 0.001)
    pot = dp.DeepPot(m, t)
    c = dp.gen_config("copper-like", 8, 8, 8, 0.1, 11)
    ro, co = O.or_compute(c, m, t)
    check(pot.compute(c), ro, pot.counters, co)


def test_list_cutoff_and_repeat_are_bitwise(cu):
    m, t, pot = cu
    c = dp.gen_config("copper-like", 5, 5, 5, 0.1, 3)
    pot.set_skin(0.0)
    a = pot.compute(c)
    pot.set_skin(2.0)
    b = pot.compute(c)
    b2 = pot.compute(c)  # reuses the buffered list
    pot.set_skin(0.0)
    assert a.energy == b.energy == b2.energy
    assert np.array_equal(a.forces, b.forces) and np.array_equal(b.forces, b2.forces)
    assert np.array_equal(a.virial, b.virial)


@pytest.mark.parametrize("seed", [500, 501, 502, 503])
def test_two_type_small_boxes(seed):
    m = dp.make_test_model(2, 6, 8, 20, 2, [18, 18], 6.0, 5.0, 401)
    t = dp.build_tables(m, 0.05)
    c = dp.make_random_config(10, 2, 9.0, 1.8, seed)
    ro, co = O.or_compute(c, m, t)
    pot = dp.DeepPot(m, t)
    check(pot.compute(c), ro, pot.counters, co)


def test_water_preset():
    m = dp.gen_model("water-like", 3)
    t = dp.build_tables(m, 0.01)
    c = dp.gen_config("water-like", 4, 4, 4, 0.1, 4)
    ro, co = O.or_compute(c, m, t)
    pot = dp.DeepPot(m, t)
    check(pot.compute(c), ro, pot.counters, co)


def test_padding_never_changes_results():
    """Slot capacity does not enter the arithmetic (test_fused.cpp:77-106): bitwise."""
    tight = dp.make_test_model(1, 6, 8, 16, 2, [8], 6.0, 5.0, 407)
    c = dp.make_random_config(10, 1, 10.0, 2.0, 73)
    L = O.or_neighbor_list(c, 6.0)
    need = int(np.max(np.diff(L.offsets)))
    tight.shape.max_nbr = [need]
    padded = tight.copy()
    padded.shape.max_nbr = [need + 40]
    t = dp.build_tables(tight, 0.01)
    pa, pb = dp.DeepPot(tight, t), dp.DeepPot(padded, t)
    a, b = pa.compute(c), pb.compute(c)
    assert a.energy == b.energy and np.array_equal(a.forces, b.forces)
    assert np.array_equal(a.virial, b.virial) and np.array_equal(a.per_atom_energy, b.per_atom_energy)
    assert pa.counters == pb.counters
    assert pa.counters.rows_forward == L.j.size


def test_extrapolation_counted():
    m = dp.make_test_model(1, 4, 6, 12, 2, [8], 6.0, 5.0, 411)
    t = dp.build_tables(m, 0.01)
    c = dp.AtomicConfig([[10, 10, 10], [10.45, 10, 10]], [0, 0], [20, 0, 0, 0, 20, 0, 0, 0, 20], [0, 0, 0])
    ro, co = O.or_compute(c, m, t)
    pot = dp.DeepPot(m, t)
    r = pot.compute(c)
    check(r, ro, pot.counters, co)
    assert pot.counters.extrapolations > 0 and np.isfinite(r.energy)


def test_overflow_and_overlap_raise_numerical_error():
    m = dp.make_test_model(1, 4, 6, 12, 2, [2], 6.0, 5.0, 417)
    t = dp.build_tables(m, 0.01)
    pot = dp.DeepPot(m, t)
    with pytest.raises(dp.NumericalError):
        pot.compute(dp.make_random_config(10, 1, 8.0, 1.8, 83))
    m = dp.make_test_model(1, 4, 6, 12, 2, [8], 6.0, 5.0, 411)
    pot = dp.DeepPot(m, dp.build_tables(m, 0.01))
    with pytest.raises(dp.NumericalError):
        pot.compute(dp.AtomicConfig([[10, 10, 10], [10, 10, 10]], [0, 0], [20, 0, 0, 0, 20, 0, 0, 0, 20], [0, 0, 0]))
    # the handle stays usable after an error
    r = pot.compute(dp.AtomicConfig([[10, 10, 10], [12, 10, 10]], [0, 0], [20, 0, 0, 0, 20, 0, 0, 0, 20], [0, 0, 0]))
    assert np.isfinite(r.energy)


def test_input_errors(cu):
    m, t, pot = cu
    c = dp.gen_config("copper-like", 3, 3, 3, 0.1, 1)
    bad = c.copy()
    bad.type[0] = 5
    with pytest.raises(dp.InputError):
        pot.compute(bad)
    bad = c.copy()
    bad.pos[0, 0] = np.nan
    with pytest.raises(dp.InputError):
        pot.compute(bad)
    bad = c.copy()
    bad.h[:] = 0
    with pytest.raises(dp.InputError):
        pot.compute(bad)


def test_finite_difference_forces_and_virial():
    """acceptance.cpp:157-222: forces by central differences, full virial vs strain."""
    m = dp.make_test_model(1, 6, 6, 16, 2, [64], 5.0, 4.0, 431)
    t = dp.build_tables(m, 0.005)
    pot = dp.DeepPot(m, t)
    c = dp.make_random_config(12, 1, 8.5, 1.8, dp.mix_seed(43, 0))
    r = pot.compute(c)
    eps = 1e-5
    fscale = max(1.0, np.max(np.abs(r.forces)))
    worst = 0.0
    for i in range(c.n_atoms):
        for x in range(3):
            up, dn = c.copy(), c.copy()
            up.pos[i, x] += eps
            dn.pos[i, x] -= eps
            fd = -(pot.compute(up).energy - pot.compute(dn).energy) / (2 * eps)
            worst = max(worst, abs(r.forces[i, x] - fd) / fscale)
    assert worst <= 1e-6
    vscale = max(1.0, np.max(np.abs(r.virial)))
    worst_v = 0.0
    for a in range(3):
        for b in range(3):
            def deformed(e):
                s = c.copy()
                h = c.h.reshape(3, 3).copy()
                h[:, a] += e * c.h.reshape(3, 3)[:, b]
                s.h = h.reshape(9).copy()
                s.pos[:, a] += e * c.pos[:, b]
                return pot.compute(s).energy
            fd = (deformed(1e-6) - deformed(-1e-6)) / 2e-6
            worst_v = max(worst_v, abs(r.virial[3 * b + a] - fd) / vscale)
    assert worst_v <= 1e-5


def test_invariances_and_force_balance():
    """acceptance.cpp:225-308: rotation + shift, relabeling, Newton's third law."""
    m = dp.make_test_model(2, 6, 6, 16, 2, [24, 24], 5.5, 4.5, 521)
    t = dp.build_tables(m, 0.01)
    pot = dp.DeepPot(m, t)
    rng = np.random.default_rng(6011)
    seedcfg = dp.make_random_config(18, 2, 8.0, 1.6, dp.mix_seed(61, 0))
    cl = dp.AtomicConfig(seedcfg.pos + 25.0, seedcfg.type, [60, 0, 0, 0, 60, 0, 0, 0, 60], [0, 0, 0])
    e0 = pot.compute(cl).energy
    for _ in range(3):
        ax = rng.normal(size=3)
        ax /= np.linalg.norm(ax)
        th = 2 * np.pi * rng.uniform()
        K = np.array([[0, -ax[2], ax[1]], [ax[2], 0, -ax[0]], [-ax[1], ax[0], 0]])
        R = np.eye(3) + np.sin(th) * K + (1 - np.cos(th)) * K @ K
        rc = cl.copy()
        rc.pos = (cl.pos - 30.0) @ R.T + 30.0 + rng.uniform(-2, 2, size=3)
        assert rel(pot.compute(rc).energy, e0) <= 1e-10
    perm = rng.permutation(cl.n_atoms)
    pc = dp.AtomicConfig(cl.pos[perm], cl.type[perm], cl.h, cl.periodic)
    assert rel(pot.compute(pc).energy, e0) <= 1e-10
    per = dp.make_random_config(16, 2, 9.0, 1.6, dp.mix_seed(62, 0))
    f = pot.compute(per).forces
    assert np.max(np.abs(f.sum(axis=0))) <= 1e-10


def test_perfect_lattice_has_zero_forces_at_scale(cu):
    """Size-independent property at a BASELINE size (C3, 1,048,576 atoms; test_io.cpp:201-216)."""
    m, t, pot = cu
    c = dp.gen_config("copper-like", 64, 64, 64, 0.0, 1)
    r = pot.compute(c)
    assert np.max(np.abs(r.forces)) <= 1e-8
    ea = r.per_atom_energy
    assert np.max(np.abs(ea - ea[0])) <= 1e-10 * abs(ea[0])
    assert rel(r.energy, ea[0] * c.n_atoms) <= 1e-10
    assert pot.counters.rows_forward == c.n_atoms * int(pot.counters.rows_forward // c.n_atoms)


def test_c3_jittered_translation_and_balance(cu):
    m, t, pot = cu
    c = dp.gen_config("copper-like", 64, 64, 64, 0.1, 11)
    a = pot.compute(c)
    s = c.copy()
    s.pos = s.pos + np.array([3.634, -2 * 3.634, 0.5])  # rigid shift (not a lattice vector)
    b = pot.compute(s)
    assert rel(a.energy, b.energy) <= 1e-10
    assert O.normwise(a.forces, b.forces) <= 1e-9
    fsum = np.abs(a.forces.sum(axis=0)).max()
    assert fsum <= 1e-9 * c.n_atoms * np.abs(a.forces).max()


def test_caller_supplied_list_matches_reference_operator(cu):
    """dp_compute_list: the reference signature compute_energy_forces_virial_tabulated(cfg, model,
    tables, list) on the reference's own list (brute path at 10 A and cell path at 8 A)."""
    m, t, pot = cu
    c = dp.gen_config("copper-like", 8, 8, 8, 0.1, 11)
    ro, co = O.or_compute(c, m, t)
    for cut, brute in ((10.0, True), (8.0, False)):
        L = O.or_neighbor_list(c, cut, brute)
        r = pot.compute_with_list(c, L)
        check(r, ro, pot.counters, co)
    # asymmetric list -> InputError, and the handle stays usable
    L = O.or_neighbor_list(c, 8.0)
    bad = dp.NeighborList(L.cutoff, L.offsets.copy(), L.j.copy(), L.shift.copy())
    bad.j[0] = (bad.j[0] + 1) % c.n_atoms
    with pytest.raises(dp.InputError):
        pot.compute_with_list(c, bad)
    check(pot.compute(c), ro, pot.counters, co)


def test_legacy_dT_kernel_matches_oracle(tmp_path):
    """The register-load k_tab_dT (fallback of the bulk-copy k_tab_dT2 for wide rows), forced by
    DPB_DT_LEGACY=1 in a fresh process (the switch is read once per process)."""
    import os
    import subprocess
    import sys
    code = r'''
import sys
sys.path.insert(0, "tests")
import oracle_lib as O
import paper_2201_01446_b200 as dp
m = dp.gen_model("copper-like", 7)
t = dp.build_tables(m, 0.01)
c = dp.gen_config("copper-like", 8, 8, 8, 0.1, 11)
ro, co = O.or_compute(c, m, t)
pot = dp.DeepPot(m, t)
r = pot.compute(c)
e = abs(r.energy - ro.energy) / abs(ro.energy)
f = O.normwise(r.forces, ro.forces)
v = O.normwise(r.virial, ro.virial)
assert max(e, f, v) <= 1e-10 and pot.counters == co, (e, f, v)
print("ok", e, f, v)
'''
    env = dict(os.environ, DPB_DT_LEGACY="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and out.stdout.startswith("ok"), out.stdout + out.stderr
