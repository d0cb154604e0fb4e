"""JSON model files: write_model / read_model (model_io.cpp:226-283), host-only (CPU).

Mirrors test_io.cpp:92-130 (bitwise round trip) plus cross-checks against the compiled reference
in both directions (our writer -> reference reader, reference writer -> our reader) and the
reference's error classes for unreadable, malformed and inconsistent files.
"""
import json

import numpy as np
import pytest

import oracle_lib as O
import paper_2201_01446_b200 as dp

needs_ref = pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref (compiled reference) not built")


@pytest.fixture(scope="module", params=["copper-like", "water-like"])
def model(request):
    return request.param, dp.gen_model(request.param, 7)


def test_round_trip_is_bitwise(tmp_path, model):
    name, m = model
    p = str(tmp_path / "m.json")
    dp.write_model(p, m, name, 7)
    mf = dp.read_model(p)
    assert mf.preset == name and mf.seed == 7
    assert mf.model.shape.n_types == m.shape.n_types
    assert mf.model.blob.tobytes() == m.blob.tobytes()
    assert (mf.model.r_cut, mf.model.r_smooth, mf.model.m_lt) == (m.r_cut, m.r_smooth, m.m_lt)
    assert mf.model.masses == m.masses and mf.model.max_nbr == m.max_nbr


@needs_ref
def test_reference_reads_our_file(tmp_path, model):
    name, m = model
    p = str(tmp_path / "ours.json")
    dp.write_model(p, m, name, 123456789012345)
    blob, seed = O.ref_read_model(p, m)
    assert seed == 123456789012345
    assert blob.tobytes() == m.blob.tobytes()


@needs_ref
def test_we_read_reference_file(tmp_path, model):
    name, m = model
    p = str(tmp_path / "ref.json")
    O.ref_write_model(p, m, name, 99)
    mf = dp.read_model(p)
    assert mf.seed == 99 and mf.preset == name
    assert mf.model.blob.tobytes() == m.blob.tobytes()
    # same document structure as the reference writes (keys, nesting)
    ours = str(tmp_path / "ours.json")
    dp.write_model(ours, m, name, 99, species=mf.species)
    a, b = json.load(open(p)), json.load(open(ours))
    assert sorted(a) == sorted(b)
    assert a["species"] == b["species"]
    assert sorted(a["fitting"][0]) == sorted(b["fitting"][0])
    assert sorted(a["embedding"][0]) == sorted(b["embedding"][0])


def test_special_values_round_trip(tmp_path):
    m = dp.make_test_model(1, 2, 2, 3, 1, [8], 6.0, 5.0, 3)
    m.blob[:6] = [0.1, -0.0, 1e-300, 5e-324, 1.7976931348623157e308, 3.0]
    p = str(tmp_path / "s.json")
    dp.write_model(p, m, "", 0)
    assert dp.read_model(p).model.blob.tobytes() == m.blob.tobytes()


@pytest.mark.parametrize("mutate,err", [
    (lambda d: d.update(format="other"), dp.InputError),
    (lambda d: d.update(version=2), dp.InputError),
    (lambda d: d.pop("masses"), dp.InputError),
    (lambda d: d["embedding"][0].update(w0=d["embedding"][0]["w0"][:-1]), dp.InputError),
    (lambda d: d.update(r_smooth=d["r_cut"]), dp.InputError),
    (lambda d: d.update(m_lt=0), dp.InputError),
    (lambda d: d["fitting"][0].update(input_width=7), dp.InputError),
    (lambda d: d.update(max_neighbors=[0] * len(d["species"])), dp.InputError),
])
def test_inconsistent_files_are_input_errors(tmp_path, mutate, err):
    m = dp.gen_model("copper-like", 7)
    p = str(tmp_path / "m.json")
    dp.write_model(p, m, "copper-like", 7)
    d = json.load(open(p))
    mutate(d)
    json.dump(d, open(p, "w"))
    with pytest.raises(err):
        dp.read_model(p)


def test_unreadable_and_malformed(tmp_path):
    with pytest.raises(dp.InputError):
        dp.read_model(str(tmp_path / "missing.json"))
    p = tmp_path / "bad.json"
    p.write_text('{"format": "dpmd-model", "version": 1,')
    with pytest.raises(dp.InputError):
        dp.read_model(str(p))
