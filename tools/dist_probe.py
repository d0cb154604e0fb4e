"""Per-rank phase timing of the domain-decomposed MD step (tools helper, not product).
  torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/dist_probe.py [rebuild_every]"""
import json, os, sys, time
from pathlib import Path
import torch, torch.distributed as dist
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2201_01446_b200 as dp

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dist.init_process_group("nccl")
rb = int(sys.argv[1]) if len(sys.argv) > 1 else 50
m = dp.gen_model("copper-like", 7); t = dp.build_tables(m, 0.01)
c = dp.gen_config("copper-like", 20 * world, 20, 20, 0.1, 11)
v = dp.init_velocities(c, m, 330.0, 99)
mc = dp.MDConfig(n_steps=1000, dt=1.0, buffer=2.0, rebuild_every=rb, thermo_every=50)
pot = dp.DeepPot(m, t, device=local)
if world > 1:
    uid = [dp.DeepPot.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    pot.dist_init(rank, world, uid[0])
pot.md_begin(c, v, mc)
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 10
pot.md_step(warm)
torch.cuda.synchronize(); dist.barrier()
pot.set_timing(True); pot.phase_times()
t0 = time.perf_counter()
pot.md_step(40)
torch.cuda.synchronize()
t1 = time.perf_counter()
ph = pot.phase_times()
out = {"rank": rank, "world": world, "rebuild_every": rb, "wall_ms_per_step": (t1 - t0) * 1e3 / 40,
       "phases_ms_per_step": {k: v[0] / 40 for k, v in ph.items()} if isinstance(next(iter(ph.values())), (list, tuple)) else {k: v / 40 for k, v in ph.items()}}
# per-step cost around the next rebuild (synchronised single steps)
per = []
for k in range(12):
    torch.cuda.synchronize(); a = time.perf_counter()
    pot.md_step(1)
    torch.cuda.synchronize(); per.append(round((time.perf_counter() - a) * 1e3, 2))
out["single_steps_ms"] = per
tag = os.environ.get("PROBE_TAG", "probe")
Path("gpurun_out").mkdir(exist_ok=True)
Path(f"gpurun_out/{tag}_r{rank}.json").write_text(json.dumps(out))
dist.barrier()
