"""Generate tests/golden/golden.json from the UNMODIFIED reference (oracle/_ref/libdpref.so).

Run here (where /root/reference exists): `python tests/golden/make_golden.py`. The fixture pins
the oracle restatement and the product's fixture generators on machines without the reference
(the GPU box). Arrays are stored as sha256 of their little-endian float64/int32 bytes plus a
few leading values; the tests recompute the hashes from the oracle.
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))
sys.path.insert(0, str(HERE.parent))

import paper_2201_01446_b200 as dp  # noqa: E402
import oracle_lib as O  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def case_eval(name, cfg, model, tabs, list_cutoff=0.0):
    r, cnt, _ = O.ref_compute(cfg, model, tabs, list_cutoff, 1)
    return {
        "name": name, "n": cfg.n_atoms, "energy": r.energy, "virial": r.virial.tolist(),
        "forces_head": r.forces[:4].tolist(), "forces_sha": sha(r.forces),
        "atom_energy_sha": sha(r.per_atom_energy), "virial_sha": sha(r.virial),
        "counters": [cnt.rows_forward, cnt.rows_backward, cnt.extrapolations],
    }


def case_list(name, cfg, cutoff):
    L = O.ref_neighbor_list(cfg, cutoff)
    return {"name": name, "cutoff": cutoff, "total": int(L.j.size), "offsets_sha": sha(L.offsets),
            "j_sha": sha(L.j), "shift_sha": sha(L.shift)}


def main() -> None:
    assert O.have_ref(), "needs oracle/_ref/libdpref.so (make -C oracle)"
    out = {"generator": "tests/golden/make_golden.py", "eval": [], "lists": [], "models": [], "md": []}
    cu = O.ref_gen_model("copper-like", 7)
    tab = O.ref_build_tables(cu, 0.01)
    out["models"].append({"name": "copper-like seed 7", "blob_sha": sha(cu.blob),
                          "tables_h0.01_sha": sha(tab.coeffs), "n_intervals": tab.n})
    wa = O.ref_gen_model("water-like", 3)
    out["models"].append({"name": "water-like seed 3", "blob_sha": sha(wa.blob),
                          "tables_h0.01_sha": sha(O.ref_build_tables(wa, 0.01).coeffs)})
    c1 = O.ref_gen_config("copper-like", 8, 8, 8, 0.1, 11)
    out["configs"] = {"C1": {"pos_sha": sha(c1.pos), "h": c1.h.tolist()}}
    out["eval"].append(case_eval("C1 Cu 8x8x8 seed 11 h 0.01", c1, cu, tab))
    out["lists"].append(case_list("C1 8A", c1, 8.0))
    out["lists"].append(case_list("C1 10A (brute path)", c1, 10.0))
    c3 = O.ref_gen_config("copper-like", 3, 3, 3, 0.1, 11)
    out["lists"].append(case_list("Cu 3x3x3 8A multi-image", c3, 8.0))
    out["eval"].append(case_eval("Cu 3x3x3 seed 11", c3, cu, tab))
    # reference test shapes (tests/test_fused.cpp, acceptance.cpp)
    shapes = [
        ("fused-equiv 2 types", (2, 6, 8, 20, 2, [18, 18], 6.0, 5.0, 401), 0.05, (10, 2, 9.0, 1.8, 500)),
        ("acceptance C3", (2, 8, 8, 20, 2, [512, 512], 5.0, 4.0, 211), 0.01, (16, 2, 9.0, 1.6, 77)),
        ("workers", (2, 6, 8, 16, 2, [14, 14], 6.0, 5.0, 413), 0.01, (17, 2, 10.0, 1.9, 79)),
    ]
    for name, margs, h, cargs in shapes:
        m = dp.make_test_model(*margs)
        blob = O.ref_make_test_model(m, margs[8])
        assert np.array_equal(blob, m.blob), name
        t = O.ref_build_tables(m, h)
        cfg = O.ref_random_config(*cargs)
        case = case_eval(name, cfg, m, t)
        case["model_args"] = margs
        case["h"] = h
        case["config_args"] = cargs
        case["model_sha"] = sha(m.blob)
        case["pos_sha"] = sha(cfg.pos)
        out["eval"].append(case)
        out["lists"].append(case_list(name + " list r_cut+1", cfg, margs[6] + 1.0))
    # short NVE run (run_md md.cpp:151-231) on Cu 3x3x3
    vel = np.empty((c3.n_atoms, 3))
    shp = cu.shape._c()
    import ctypes as C
    O._chk(O.ref().ref_init_velocities(C.byref(shp), c3.n_atoms, dp._dp(c3.pos), dp._ip(c3.type),
                                       dp._dp(c3.h), 330.0, 99, dp._dp(vel)), O.ref(), "ref_last_error")
    v0 = vel.copy()
    cfg = c3.copy()
    mc = dp.MDConfig(n_steps=20, dt=1.0, buffer=2.0, rebuild_every=10, thermo_every=5)
    res = O.ref_run_md(cfg, vel, cu, tab, mc)
    out["md"].append({
        "name": "Cu 3x3x3 NVE 20 steps", "vel0_sha": sha(v0), "thermo": [[t.step, t.ke, t.pe, t.temperature, t.pressure] for t in res.thermo],
        "force_evals": res.force_evals, "staleness_checks": res.staleness_checks,
        "final_total": res.final_total, "pos_sha": sha(cfg.pos), "vel_sha": sha(vel),
        "counters": [res.counters.rows_forward, res.counters.rows_backward, res.counters.extrapolations],
    })
    (HERE / "golden.json").write_text(json.dumps(out, indent=1))
    print("wrote", HERE / "golden.json")


if __name__ == "__main__":
    main()
