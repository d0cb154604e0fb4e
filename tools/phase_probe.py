"""Phase times of repeated C2 evaluations (tools helper, not product)."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2201_01446_b200 as dp
prec = sys.argv[1] if len(sys.argv) > 1 else "fp64"
m = dp.gen_model("copper-like", 7); t = dp.build_tables(m, 0.01)
c = dp.gen_config("copper-like", 20, 20, 20, 0.1, 11)
pot = dp.DeepPot(m, t, precision=prec)
pot.set_skin(2.0)
for _ in range(3): pot.compute(c)
pot.set_timing(True); pot.phase_times()
for _ in range(10): pot.compute(c)
ph = pot.phase_times()
print(json.dumps({k: round(v[0] / 10, 4) for k, v in ph.items()}))
