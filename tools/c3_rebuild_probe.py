"""Per-step times of a 1 M-atom (C3) MD run around the list rebuilds (tools helper, not product);
run with DPB_TRACE=1 to see the allocations of each rebuild."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2201_01446_b200 as dp
m = dp.gen_model("copper-like", 7)
t = dp.build_tables(m, 0.01)
c = dp.gen_config("copper-like", 64, 64, 64, 0.1, 11)
v = dp.init_velocities(c, m, 330.0, 99)
pot = dp.DeepPot(m, t)
pot.md_begin(c, v, dp.MDConfig(n_steps=160, dt=1.0, buffer=2.0, rebuild_every=50, thermo_every=10 ** 9))
st = torch.cuda.ExternalStream(pot.stream)
for k in range(1, 151):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(st); h0 = time.perf_counter(); pot.md_step(1); h1 = time.perf_counter(); b.record(st); b.synchronize()
    ms = a.elapsed_time(b)
    if k % 50 == 0 or k % 50 == 1 or ms > 160:
        print("step", k, "gpu ms %.1f host ms %.1f" % (ms, (h1 - h0) * 1e3), flush=True)
pot.md_end()
