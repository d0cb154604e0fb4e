"""Per-step CUDA-event times of the C2 MD loop (tools helper): finds stalls inside the loop."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2201_01446_b200 as dp

m = dp.gen_model("copper-like", 7)
t = dp.build_tables(m, 0.01)
c = dp.gen_config("copper-like", 20, 20, 20, 0.1, 11)
v = dp.init_velocities(c, m, 330.0, 99)
pot = dp.DeepPot(m, t)
N = int(sys.argv[1]) if len(sys.argv) > 1 else 160
pot.md_begin(c, v, dp.MDConfig(n_steps=N + 10, dt=1.0, buffer=2.0, rebuild_every=50, thermo_every=10 ** 9))
st = torch.cuda.ExternalStream(pot.stream)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(N + 1)]
host = []
ev[0].record(st)
for k in range(N):
    h0 = time.perf_counter()
    pot.md_step(1)
    host.append(time.perf_counter() - h0)
    ev[k + 1].record(st)
ev[-1].synchronize()
ms = np.array([ev[k].elapsed_time(ev[k + 1]) for k in range(N)])
print("median %.3f  mean %.3f  max %.3f at step %d" % (np.median(ms), ms.mean(), ms.max(), ms.argmax() + 1))
slow = [(k + 1, round(ms[k], 3), round(host[k] * 1e3, 3)) for k in range(N) if ms[k] > 1.2 * np.median(ms)]
print("slow steps (step, gpu ms, host ms):", slow)
print("host ms median %.3f max %.3f" % (np.median(host) * 1e3, max(host) * 1e3))
pot.md_end()
