"""Device-resident velocity Verlet (run_md md.cpp:151-231) against the oracle and the reference's
MD tests (test_domain_md.cpp:184-319, acceptance.cpp C7/C9)."""
import json
from pathlib import Path

import numpy as np
import pytest

import oracle_lib as O
import paper_2201_01446_b200 as dp

pytestmark = pytest.mark.gpu
GOLDEN = json.loads((Path(__file__).parent / "golden" / "golden.json").read_text())


def test_md_matches_reference_golden():
    m = dp.gen_model("copper-like", 7)
    t = dp.build_tables(m, 0.01)
    c = dp.gen_config("copper-like", 3, 3, 3, 0.1, 11)
    v = dp.init_velocities(c, m, 330.0, 99)
    res = dp.DeepPot(m, t).run_md(c, v, dp.MDConfig(n_steps=20, dt=1.0, buffer=2.0, rebuild_every=10, thermo_every=5))
    g = GOLDEN["md"][0]
    assert res.force_evals == g["force_evals"] and res.staleness_checks == g["staleness_checks"]
    assert [r.step for r in res.thermo] == [x[0] for x in g["thermo"]]
    for r, x in zip(res.thermo, g["thermo"]):
        assert abs(r.pe - x[2]) <= 1e-10 * abs(x[2])
        assert abs(r.ke - x[1]) <= 1e-9 * abs(x[1])
        assert abs(r.pressure - x[4]) <= 1e-8 * abs(x[4])
    assert abs(res.final_total - g["final_total"]) <= 1e-10 * abs(g["final_total"])
    assert [res.counters.rows_forward, res.counters.rows_backward, res.counters.extrapolations] == g["counters"]


def test_md_matches_oracle_two_types():
    m = dp.make_test_model(2, 5, 6, 14, 2, [24, 24], 5.5, 4.5, 811)
    t = dp.build_tables(m, 0.01)
    base = dp.make_random_config(16, 2, 10.0, 2.0, 811)
    mc = dp.MDConfig(n_steps=30, dt=1.0, rebuild_every=10, thermo_every=10)
    c1, c2 = base.copy(), base.copy()
    v1 = dp.init_velocities(c1, m, 250.0, 13)
    v2 = v1.copy()
    a = dp.DeepPot(m, t).run_md(c1, v1, mc)
    b = O.or_run_md(c2, v2, m, t, mc)
    assert a.force_evals == b.force_evals == 31
    for x, y in zip(a.thermo, b.thermo):
        assert x.step == y.step
        assert abs(x.pe - y.pe) <= 1e-9 * max(1.0, abs(y.pe))
    assert O.normwise(c1.pos, c2.pos) <= 1e-10
    assert O.normwise(v1, v2) <= 1e-8


def test_99_steps_is_100_evaluations_and_thermo_cadence():
    m = dp.make_test_model(1, 4, 6, 12, 2, [16], 5.0, 4.0, 947)
    t = dp.build_tables(m, 0.01)
    c = dp.make_random_config(8, 1, 9.0, 2.2, 97)
    v = dp.init_velocities(c, m, 50.0, 7)
    pot = dp.DeepPot(m, t)
    res = pot.run_md(c, v, dp.MDConfig(n_steps=99, thermo_every=50))
    assert res.force_evals == 100 and res.staleness_checks == 99
    assert [r.step for r in res.thermo] == [0, 50]
    c2 = dp.make_random_config(8, 1, 9.0, 2.2, 98)
    v2 = dp.init_velocities(c2, m, 50.0, 7)
    res = pot.run_md(c2, v2, dp.MDConfig(n_steps=0))
    assert res.force_evals == 1 and len(res.thermo) == 1


def test_first_pe_equals_direct_evaluation():
    m = dp.make_test_model(2, 5, 6, 14, 2, [12, 12], 5.5, 4.5, 963)
    t = dp.build_tables(m, 0.01)
    c = dp.make_random_config(14, 2, 10.0, 2.0, 103)
    pot = dp.DeepPot(m, t)
    direct = pot.compute(c).energy
    v = dp.init_velocities(c, m, 200.0, 17)
    res = pot.run_md(c.copy(), v, dp.MDConfig(n_steps=0, buffer=2.0))
    assert res.thermo[0].pe == direct


def test_stale_list_aborts_and_rebuild_every_step_survives():
    m = dp.make_test_model(1, 4, 6, 12, 2, [8], 6.0, 5.0, 953)
    t = dp.build_tables(m, 0.05)
    box = [100, 0, 0, 0, 100, 0, 0, 0, 100]
    pot = dp.DeepPot(m, t)
    c = dp.AtomicConfig([[20, 50, 50], [80, 50, 50]], [0, 0], box, [0, 0, 0])
    v = dp.init_velocities(c, m, 2000.0, 11)
    with pytest.raises(dp.NumericalError):
        pot.run_md(c, v, dp.MDConfig(n_steps=50, dt=1.0, buffer=0.01, rebuild_every=1000))
    c = dp.AtomicConfig([[20, 50, 50], [80, 50, 50]], [0, 0], box, [0, 0, 0])
    v = dp.init_velocities(c, m, 2000.0, 11)
    res = pot.run_md(c, v, dp.MDConfig(n_steps=50, dt=1.0, buffer=0.01, rebuild_every=1))
    assert res.force_evals == 51


def test_nve_energy_conservation_fine_table():
    """Acceptance C7 shape (acceptance.cpp:330-358), 200 steps instead of 1000."""
    p = dp.get_preset("copper-like")
    m = dp.gen_model(p, 7)
    t = dp.build_tables(m, 0.001)
    c = dp.gen_config(p, 3, 3, 3, 0.1, 11)
    v = dp.init_velocities(c, m, 330.0, 99)
    res = dp.DeepPot(m, t).run_md(c, v, dp.MDConfig(n_steps=200, dt=1.0, buffer=2.0, rebuild_every=50, thermo_every=1))
    e0 = res.thermo[0].ke + res.thermo[0].pe
    drift = max(abs(r.ke + r.pe - e0) for r in res.thermo)
    mean_ke = np.mean([r.ke for r in res.thermo])
    assert drift <= 1e-4 * mean_ke
    assert res.staleness_checks == 200 and res.max_drift_seen <= 1.0


def test_md_step_past_configured_count_is_input_error():
    """dp_md_step beyond MDConfig.n_steps must not run past the thermo buffer."""
    m = dp.make_test_model(1, 4, 6, 12, 2, [16], 5.0, 4.0, 947)
    t = dp.build_tables(m, 0.01)
    c = dp.make_random_config(8, 1, 9.0, 2.2, 97)
    v = dp.init_velocities(c, m, 50.0, 7)
    pot = dp.DeepPot(m, t)
    pot.md_begin(c, v, dp.MDConfig(n_steps=5, thermo_every=1))
    pot.md_step(3)
    with pytest.raises(dp.InputError):
        pot.md_step(3)
    pot.md_step(2)
    res = pot.md_end()
    assert res.force_evals == 6 and [r.step for r in res.thermo] == list(range(6))
