"""Host enqueue time and device time per MD step (tools helper, not product)."""
import json, sys, time
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2201_01446_b200 as dp
prec = sys.argv[1] if len(sys.argv) > 1 else "fp64"
timing = len(sys.argv) > 2 and sys.argv[2] == "timing"
m = dp.gen_model("copper-like", 7); t = dp.build_tables(m, 0.01)
c = dp.gen_config("copper-like", 20, 20, 20, 0.1, 11)
v = dp.init_velocities(c, m, 330.0, 99)
mc = dp.MDConfig(n_steps=1000, dt=1.0, buffer=2.0, rebuild_every=50, thermo_every=10**9)
pot = dp.DeepPot(m, t, precision=prec)
pot.md_begin(c, v, mc)
pot.md_step(10)
st = torch.cuda.ExternalStream(pot.stream)
torch.cuda.synchronize()
if timing:
    pot.set_timing(True); pot.phase_times()
host, evs = [], []
for k in range(100):
    e = torch.cuda.Event(enable_timing=True); e.record(st); evs.append(e)
    a = time.perf_counter(); pot.md_step(1); host.append((time.perf_counter() - a) * 1e3)
e = torch.cuda.Event(enable_timing=True); e.record(st); evs.append(e)
torch.cuda.synchronize()
dev = [evs[k].elapsed_time(evs[k + 1]) for k in range(100)]
big = [(k + 11, round(host[k], 2), round(dev[k], 2)) for k in range(100) if host[k] > 1.0 or dev[k] > 7.0]
print(json.dumps({"prec": prec, "timing": timing, "dev_total_ms": round(sum(dev), 2), "median_dev": sorted(dev)[50],
                  "outliers(step,host_ms,dev_ms)": big}))
