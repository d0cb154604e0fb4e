"""Host-side cost of the e2e loop at C2: dp_compute alone, numpy and torch host integrators (tools helper)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2201_01446_b200 as dp
m = dp.gen_model("copper-like", 7); t = dp.build_tables(m, 0.01)
c = dp.gen_config("copper-like", 20, 20, 20, 0.1, 11)
n = c.n_atoms
pin = lambda shape: torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()
pot = dp.DeepPot(m, t); pot.set_skin(2.0)
c2 = dp.AtomicConfig(c.pos, c.type, c.h); pos = pin((n, 3)); pos[:] = c.pos; c2.pos = pos
f = pin((n, 3)); v = pin((n, 3)); v[:] = 1e-4
r = pot.compute(c2, forces_out=f)
for k in range(5): pot.compute(c2, forces_out=f)
K = 30
t0 = time.perf_counter()
for k in range(K): pot.compute(c2, forces_out=f)
t1 = time.perf_counter()
for k in range(K):
    v += 0.5 * f * 1e-6; pos += v; v += 0.5 * f * 1e-6
t2 = time.perf_counter()
print("compute only %.3f ms/call, numpy verlet %.3f ms/step" % ((t1 - t0) / K * 1e3, (t2 - t1) / K * 1e3))
import cProfile, pstats
cProfile.run("for k in range(10): pot.compute(c2, forces_out=f)", "/tmp/prof")
pstats.Stats("/tmp/prof").sort_stats("cumtime").print_stats(8)
tv, tf, tp = torch.from_numpy(v), torch.from_numpy(f), torch.from_numpy(pos)
t3 = time.perf_counter()
for k in range(K):
    tp.add_(tv); tv.add_(tf, alpha=1e-6)
t4 = time.perf_counter()
print("torch leapfrog %.3f ms/step (threads %d)" % ((t4 - t3) / K * 1e3, torch.get_num_threads()))
