"""Per-rank, per-step CUDA-event times of the weak-scaled C2 MD loop (tools helper, not product).

usage: python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/step_times_dist.py [steps]
Prints, per rank, the median / max step and the steps slower than 1.2x the median (host time of
the md_step call beside it), to locate stalls that inflate one rank's window.
"""
import os
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch
import torch.distributed as dist

import paper_2201_01446_b200 as dp

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
m = dp.gen_model("copper-like", 7)
t = dp.build_tables(m, 0.01)
c = dp.gen_config("copper-like", 20 * world, 20, 20, 0.1, 11)
v = dp.init_velocities(c, m, 330.0, 99)
pot = dp.DeepPot(m, t, device=local)
uid = [dp.DeepPot.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(uid, src=0)
pot.dist_init(rank, world, uid[0])
N = int(sys.argv[1]) if len(sys.argv) > 1 else 120
pot.md_begin(c, v, dp.MDConfig(n_steps=N + 20, dt=1.0, buffer=2.0, rebuild_every=50, thermo_every=10 ** 9))
pot.md_step(10)
st = torch.cuda.ExternalStream(pot.stream, device=torch.device("cuda", local))
torch.cuda.synchronize()
dist.barrier()
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
slow = [(k + 11, round(float(ms[k]), 3), round(host[k] * 1e3, 3)) for k in range(N) if ms[k] > 1.2 * np.median(ms)]
for r in range(world):
    if r == rank:
        print(f"rank {rank}: total {ms.sum():.2f} ms  median {np.median(ms):.3f}  max {ms.max():.3f} at step "
              f"{ms.argmax() + 11}; slow (step, gpu ms, host ms): {slow}", flush=True)
    dist.barrier()
pot.md_end()
dist.destroy_process_group()
