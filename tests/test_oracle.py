"""The CPU oracle (oracle/dp_oracle.cpp) is pinned to the reference: golden vectors and, where
oracle/_ref exists, bitwise equality with the live reference library."""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

import oracle_lib as O
import paper_2201_01446_b200 as dp

GOLDEN = json.loads((Path(__file__).parent / "golden" / "golden.json").read_text())
needs_ref = pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built (no /root/reference)")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def golden_case(name):
    return next(c for c in GOLDEN["eval"] if c["name"].startswith(name))


@pytest.fixture(scope="module")
def cu():
    m = dp.gen_model("copper-like", 7)
    return m, dp.build_tables(m, 0.01)


def check_eval(r, cnt, g):
    assert r.energy == g["energy"]
    assert sha(r.forces) == g["forces_sha"]
    assert sha(r.per_atom_energy) == g["atom_energy_sha"]
    assert sha(r.virial) == g["virial_sha"]
    assert [cnt.rows_forward, cnt.rows_backward, cnt.extrapolations] == g["counters"]


def test_oracle_c1_golden(cu):
    m, t = cu
    c = dp.gen_config("copper-like", 8, 8, 8, 0.1, 11)
    r, cnt = O.or_compute(c, m, t)
    check_eval(r, cnt, golden_case("C1"))
    # the survey's golden numbers
    assert r.energy == -322.55577501639613
    assert abs(r.virial[0] + r.virial[4] + r.virial[8] - (-1219.6869569938162)) < 1e-9


def test_oracle_small_cases_golden():
    for g in GOLDEN["eval"]:
        if "model_args" not in g:
            continue
        m = dp.make_test_model(*g["model_args"])
        t = dp.build_tables(m, g["h"])
        c = dp.make_random_config(*g["config_args"])
        r, cnt = O.or_compute(c, m, t)
        check_eval(r, cnt, g)


def test_oracle_lists_golden():
    c1 = dp.gen_config("copper-like", 8, 8, 8, 0.1, 11)
    c3 = dp.gen_config("copper-like", 3, 3, 3, 0.1, 11)
    cases = {"C1 8A": (c1, 8.0), "C1 10A (brute path)": (c1, 10.0), "Cu 3x3x3 8A multi-image": (c3, 8.0)}
    for g in GOLDEN["lists"]:
        if g["name"] not in cases:
            continue
        c, cut = cases[g["name"]]
        L = O.or_neighbor_list(c, cut)
        assert L.j.size == g["total"]
        assert sha(L.offsets) == g["offsets_sha"] and sha(L.j) == g["j_sha"] and sha(L.shift) == g["shift_sha"]


def test_oracle_md_golden(cu):
    m, t = cu
    g = GOLDEN["md"][0]
    c = dp.gen_config("copper-like", 3, 3, 3, 0.1, 11)
    v = dp.init_velocities(c, m, 330.0, 99)
    assert sha(v) == g["vel0_sha"]
    res = O.or_run_md(c, v, m, t, dp.MDConfig(n_steps=20, dt=1.0, buffer=2.0, rebuild_every=10, thermo_every=5))
    assert [[r.step, r.ke, r.pe, r.temperature, r.pressure] for r in res.thermo] == g["thermo"]
    assert res.force_evals == g["force_evals"] == 21
    assert res.staleness_checks == g["staleness_checks"]
    assert res.final_total == g["final_total"]
    assert sha(c.pos) == g["pos_sha"] and sha(v) == g["vel_sha"]


@needs_ref
@pytest.mark.parametrize("seed", [42, 43])
def test_oracle_lists_live_reference_multi_image(seed):
    c = dp.make_random_config(12, 2, 6.0, 1.0, seed)  # box 6 < cutoff 7: several images
    assert O.lists_equal(O.or_neighbor_list(c, 7.0), O.ref_neighbor_list(c, 7.0))
    c = dp.make_random_config(120, 2, 30.0, 1.2, seed)  # cell path
    assert O.lists_equal(O.or_neighbor_list(c, 5.0), O.ref_neighbor_list(c, 5.0))
    assert O.lists_equal(O.or_neighbor_list(c, 5.0, brute=True), O.ref_neighbor_list(c, 5.0, brute=True))


@needs_ref
def test_oracle_live_reference_water():
    m = dp.gen_model("water-like", 3)
    t = dp.build_tables(m, 0.01)
    c = dp.gen_config("water-like", 3, 3, 3, 0.1, 4)
    r, cnt = O.or_compute(c, m, t, 8.0)
    rr, cr, _ = O.ref_compute(c, m, t, 8.0, 2)
    assert r.energy == rr.energy and np.array_equal(r.forces, rr.forces)
    assert np.array_equal(r.virial, rr.virial) and cnt == cr


def test_oracle_overflow_and_overlap_raise():
    m = dp.make_test_model(1, 4, 6, 12, 2, [2], 6.0, 5.0, 417)
    t = dp.build_tables(m, 0.01)
    c = dp.make_random_config(10, 1, 8.0, 1.8, 83)
    with pytest.raises(dp.NumericalError):
        O.or_compute(c, m, t)
    m = dp.make_test_model(1, 4, 6, 12, 2, [8], 6.0, 5.0, 411)
    t = dp.build_tables(m, 0.01)
    c = dp.AtomicConfig([[10, 10, 10], [10, 10, 10]], [0, 0], [20, 0, 0, 0, 20, 0, 0, 0, 20], [0, 0, 0])
    with pytest.raises(dp.NumericalError):
        O.or_compute(c, m, t)
