"""The paper's 13.5 M-atom copper system (BASELINE config C4) on ONE B200 (VERDICT r01 "Next #7").

A full reference evaluation of C4 takes over an hour of host CPU, so parity is checked through
properties that do not depend on the system size:
  * locality: E_i and F_i of interior atoms equal the reference's values for a non-periodic
    cluster holding every atom within 2 r_c + 1 A of them (E_i depends on atoms within r_c,
    F_i on atoms within 2 r_c) -- compute_energy_forces_virial_tabulated on the cluster;
  * force balance: sum_i F_i = 0 to rounding (exact.cpp:22-38 scatters +g / -g per pair);
  * counters: rows_forward == rows_backward, no extrapolation.
"""
import numpy as np
import pytest

import oracle_lib as O
import paper_2201_01446_b200 as dp

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.mark.timeout(1800)
def test_c4_single_gpu_locality_and_balance():
    m = dp.gen_model("copper-like", 7)
    t = dp.build_tables(m, 0.01)
    c = dp.gen_config("copper-like", 150, 150, 150, 0.1, 11)
    assert c.n_atoms == 13_500_000
    pot = dp.DeepPot(m, t)
    r = pot.compute(c)
    cnt = pot.counters
    pot.close()
    assert cnt.rows_forward == cnt.rows_backward and cnt.extrapolations == 0
    assert 175.0 < cnt.rows_forward / c.n_atoms < 180.0
    fmax = float(np.max(np.abs(r.forces)))
    # force balance: |sum F| at the rounding level of 13.5 M terms of size fmax
    assert float(np.max(np.abs(r.forces.sum(axis=0)))) <= 1e-12 * fmax * c.n_atoms
    assert abs(r.energy - r.per_atom_energy.sum()) <= 1e-12 * abs(r.energy)
    box = c.h.reshape(3, 3).diagonal()
    rad = 2.0 * m.r_cut + 1.0
    rng = np.random.default_rng(5)
    picks = rng.choice(c.n_atoms, 64, replace=False)
    interior = [i for i in picks if np.all(c.pos[i] > rad + 1.0) and np.all(c.pos[i] < box - rad - 1.0)][:4]
    assert len(interior) >= 3
    for i in interior:
        near = np.nonzero(np.sum((c.pos - c.pos[i]) ** 2, axis=1) <= rad * rad)[0]
        k = int(np.searchsorted(near, i))
        L = 4.0 * rad + 50.0
        cl = dp.AtomicConfig(c.pos[near] - c.pos[i] + L / 2, c.type[near], [L, 0, 0, 0, L, 0, 0, 0, L], [0, 0, 0])
        ro, _, _ = O.ref_compute(cl, m, t, 0.0, 16)
        assert abs(r.per_atom_energy[i] - ro.per_atom_energy[k]) <= 1e-10 * abs(ro.per_atom_energy[k])
        assert float(np.max(np.abs(r.forces[i] - ro.forces[k]))) <= 1e-10 * fmax
