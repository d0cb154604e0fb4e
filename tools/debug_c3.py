import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2201_01446_b200 as dp, oracle_lib as O
cells = int(sys.argv[1])
m = dp.gen_model("copper-like", 7); t = dp.build_tables(m, 0.01)
cp = dp.gen_config("copper-like", cells, cells, cells, 0.0, 1)
cj = dp.gen_config("copper-like", cells, cells, cells, 0.1, 11)
fresh = dp.DeepPot(m, t)
rf = fresh.compute(cj)
pot = dp.DeepPot(m, t)
pot.compute(cp)
try:
    rj = pot.compute(cj)
    print(cells, "after-perfect vs fresh: dF", O.normwise(rj.forces, rf.forces), "dE", abs(rj.energy - rf.energy), flush=True)
except Exception as e:
    print(cells, "raised", type(e).__name__, e, flush=True)
