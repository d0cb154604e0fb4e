"""Forward contraction from a staged 32-centre interval union (DPB_T2=1: k_tab_fwd<WM> moments +
k_tab_fwd_T2, tabulate.cu). Run in a subprocess because the switch is read once per process.
Checks: bitwise equal to the per-warp k_tab_fwd path (same FMA chain per accumulator), within
1e-10 of the oracle, counters equal, and bitwise independent of the chunking,
including chunk sizes that shift the 32-centre block boundaries."""
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import oracle_lib as O
import paper_2201_01446_b200 as dp

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2201_01446_b200 as dp
m = dp.gen_model("copper-like", 7); t = dp.build_tables(m, 0.01)
c = dp.gen_config("copper-like", 8, 8, 8, 0.1, 11)
out = {}
for ch in (0, 100, 333):
    pot = dp.DeepPot(m, t)
    if ch: pot.set_chunk_size(ch)
    r = pot.compute(c)
    k = pot.counters
    ctr = [k.rows_forward, k.rows_backward, k.extrapolations]
    r2 = pot.compute(c)  # second evaluation: Pbuf sized, no count pass
    assert r2.energy == r.energy and np.array_equal(r2.forces, r.forces)
    out[ch] = {"e": r.energy, "f": r.forces.tolist(), "v": r.virial.tolist(),
               "ae": r.per_atom_energy.tolist(), "ctr": ctr}
print(json.dumps(out))
"""


def test_t2_forward_parity_and_chunk_bitwise():
    env = dict(os.environ, DPB_T2="1")
    p = subprocess.run([sys.executable, "-c", SCRIPT, str(ROOT)], env=env, capture_output=True, text=True,
                       timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    out = json.loads(p.stdout.strip().splitlines()[-1])
    base = out["0"]
    for k in ("100", "333"):
        assert out[k] == base  # bitwise: same floats after the JSON round trip
    m = dp.gen_model("copper-like", 7)
    t = dp.build_tables(m, 0.01)
    c = dp.gen_config("copper-like", 8, 8, 8, 0.1, 11)
    ref = dp.DeepPot(m, t).compute(c)  # this process: the per-warp forward kernel
    assert base["e"] == ref.energy
    assert np.array_equal(np.array(base["f"]), ref.forces)
    assert np.array_equal(np.array(base["v"]), ref.virial)
    assert np.array_equal(np.array(base["ae"]), ref.per_atom_energy)
    ro, co = O.or_compute(c, m, t)
    assert abs(base["e"] - ro.energy) <= 1e-10 * abs(ro.energy)
    assert O.normwise(np.array(base["f"]), ro.forces) <= 1e-10
    assert O.normwise(np.array(base["v"]), ro.virial) <= 1e-10
    assert O.normwise(np.array(base["ae"]), ro.per_atom_energy) <= 1e-10
    assert base["ctr"] == [co.rows_forward, co.rows_backward, co.extrapolations]
