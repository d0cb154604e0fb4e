"""Mixed-precision error budget probe (tools helper): E/F/V/E_i errors of precision='mixed' against
the FP64 oracle on the presets of tests/test_gpu_mixed.py (run with/without DPB_MIXED_TAB64=1)."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import oracle_lib as O
import paper_2201_01446_b200 as dp

def metrics(r, ro):
    return {"E": abs(r.energy - ro.energy) / abs(ro.energy), "F": O.normwise(r.forces, ro.forces),
            "V": O.normwise(r.virial, ro.virial), "Ei": O.normwise(r.per_atom_energy, ro.per_atom_energy)}

cases = []
m = dp.gen_model("water-like", 3); t = dp.build_tables(m, 0.01); c = dp.gen_config("water-like", 4, 4, 4, 0.1, 4)
cases.append(("water", m, t, c))
m = dp.make_test_model(2, 6, 8, 20, 2, [18, 18], 6.0, 5.0, 401); t = dp.build_tables(m, 0.05)
cases.append(("two_type", m, t, dp.make_random_config(10, 2, 9.0, 1.8, 500)))
m = dp.gen_model("copper-like", 7); t = dp.build_tables(m, 0.01)
cases.append(("cu_c1", m, t, dp.gen_config("copper-like", 8, 8, 8, 0.1, 11)))
for name, m, t, c in cases:
    ro, _ = O.or_compute(c, m, t)
    r = dp.DeepPot(m, t, precision="mixed").compute(c)
    print(name, {k: f"{v:.2e}" for k, v in metrics(r, ro).items()}, "E", ro.energy, flush=True)
