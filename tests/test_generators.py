"""Host-side fixture generators are bit-identical to the reference (golden hashes + live _ref)."""
import hashlib
import json
import math
from pathlib import Path

import numpy as np
import pytest

import oracle_lib as O
import paper_2201_01446_b200 as dp

GOLDEN = json.loads((Path(__file__).parent / "golden" / "golden.json").read_text())
needs_ref = pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built (no /root/reference)")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_copper_model_tables_config_match_golden():
    m = dp.gen_model("copper-like", 7)
    g = GOLDEN["models"][0]
    assert sha(m.blob) == g["blob_sha"]
    t = dp.build_tables(m, 0.01)
    assert t.n == g["n_intervals"] == 200
    assert sha(t.coeffs) == g["tables_h0.01_sha"]
    c = dp.gen_config("copper-like", 8, 8, 8, 0.1, 11)
    assert sha(c.pos) == GOLDEN["configs"]["C1"]["pos_sha"]
    assert c.h.tolist() == GOLDEN["configs"]["C1"]["h"]


def test_water_model_and_tables_match_golden():
    m = dp.gen_model("water-like", 3)
    g = GOLDEN["models"][1]
    assert sha(m.blob) == g["blob_sha"]
    assert sha(dp.build_tables(m, 0.01).coeffs) == g["tables_h0.01_sha"]


def test_test_models_match_golden():
    for case in GOLDEN["eval"]:
        if "model_args" not in case:
            continue
        m = dp.make_test_model(*case["model_args"])
        assert sha(m.blob) == case["model_sha"], case["name"]
        c = dp.make_random_config(*case["config_args"])
        assert sha(c.pos) == case["pos_sha"], case["name"]


@needs_ref
@pytest.mark.parametrize("preset,seed", [("copper-like", 1), ("water-like", 5)])
def test_gen_model_live_reference(preset, seed):
    assert np.array_equal(dp.gen_model(preset, seed).blob, O.ref_gen_model(preset, seed).blob)


@needs_ref
@pytest.mark.parametrize("h", [0.1, 0.05, 0.003])
def test_build_tables_live_reference(h):
    m = dp.make_test_model(2, 5, 4, 12, 2, [8, 8], 6.0, 5.0, 303)
    assert np.array_equal(dp.build_tables(m, h).coeffs, O.ref_build_tables(m, h).coeffs)


@needs_ref
def test_configs_live_reference():
    a = dp.gen_config("water-like", 3, 2, 4, 0.2, 5)
    b = O.ref_gen_config("water-like", 3, 2, 4, 0.2, 5)
    assert np.array_equal(a.pos, b.pos) and np.array_equal(a.type, b.type)
    a = dp.make_random_config(24, 3, 10.0, 1.4, 871)
    b = O.ref_random_config(24, 3, 10.0, 1.4, 871)
    assert np.array_equal(a.pos, b.pos) and np.array_equal(a.type, b.type)


def test_table_domain_and_interval_count():
    # table_domain_end = s(0.5 A) = 2.0 for the copper preset (test_table.cpp:157-167)
    m = dp.gen_model("copper-like", 7)
    t = dp.build_tables(m, 0.01)
    assert t.x_end() == pytest.approx(2.0, abs=1e-12)
    t = dp.build_tables(m, 0.001)
    assert t.n == 2000


def test_dptb_round_trip(tmp_path):
    m = dp.make_test_model(2, 4, 4, 12, 2, [8, 8], 6.0, 5.0, 9)
    t = dp.build_tables(m, 0.05)
    p = tmp_path / "t.dptb"
    dp.write_tables(str(p), t)
    raw = p.read_bytes()
    assert raw[:4] == b"DPTB"
    u = dp.read_tables(str(p))
    assert (u.n, u.m, u.block, u.x0, u.h) == (t.n, t.m, t.block, t.x0, t.h)
    assert np.array_equal(u.coeffs, t.coeffs)
    bad = tmp_path / "bad.dptb"
    bad.write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(dp.InputError):
        dp.read_tables(str(bad))
    short = tmp_path / "short.dptb"
    short.write_bytes(raw[: len(raw) // 2])
    with pytest.raises(dp.InputError):
        dp.read_tables(str(short))


def test_init_velocities_properties():
    m = dp.gen_model("copper-like", 7)
    c = dp.gen_config("copper-like", 3, 3, 3, 0.1, 11)
    v = dp.init_velocities(c, m, 330.0, 99)
    mass = 63.546
    assert np.allclose(v.sum(axis=0) * mass, 0.0, atol=1e-12)
    mvv = 1.0e7 / (6.02214076e23 * 1.602176634e-19)
    ke = 0.5 * mass * (v * v).sum() * mvv
    t = 2 * ke / (3 * c.n_atoms * 8.617333262e-5)
    assert t == pytest.approx(330.0, rel=1e-12)


def tanh_eval(coef, x):
    ax = abs(x)
    if ax > 8.0:
        t = 1.0
    else:
        k = int(ax * 1024.0)
        u = ax - k * (1.0 / 1024.0)
        c = coef[k]
        t = c[0] + u * (c[1] + u * c[2])
    return -t if math.copysign(1.0, x) < 0 else t


def test_tanh_table_accuracy():
    """Acceptance C6 (acceptance.cpp:311-327) on the product's table coefficients."""
    coef = dp.tanh_table()
    xs = np.linspace(-8.0, 8.0, 20001)
    worst = max(abs(tanh_eval(coef, float(x)) - math.tanh(float(x))) for x in xs)
    assert worst <= 1.2e-7
    assert tanh_eval(coef, 8.5) == 1.0 and tanh_eval(coef, -1e300) == -1.0 and tanh_eval(coef, 0.0) == 0.0
    assert all(tanh_eval(coef, -float(x)) == -tanh_eval(coef, float(x)) for x in xs[::97])
