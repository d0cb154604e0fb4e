"""Distributed MD (torchrun, one rank per GPU) vs the single-GPU path on the same global system.

  torchrun --nproc-per-node N --master-addr 127.0.0.1 tests/dist/dist_md_check.py [out.json]
Rank 0 writes a JSON verdict. Used by tests/test_gpu_dist.py (needs >= 2 GPUs).
"""
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_2201_01446_b200 as dp  # noqa: E402


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl")
    m = dp.gen_model("copper-like", 7)
    t = dp.build_tables(m, 0.01)
    c = dp.gen_config("copper-like", 7 * world, 6, 6, 0.1, 11)
    v = dp.init_velocities(c, m, 330.0, 99)
    mc = dp.MDConfig(n_steps=60, dt=1.0, buffer=2.0, rebuild_every=20, thermo_every=10)
    pot = dp.DeepPot(m, t, device=local)
    uid = [dp.DeepPot.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    pot.dist_init(rank, world, uid[0])
    cd, vd = c.copy(), v.copy()
    pot.md_begin(cd, vd, mc)
    pot.md_step(mc.n_steps)
    pos = np.empty_like(c.pos)
    vel = np.empty_like(v)
    rd = pot.md_end(pos, vel)
    dist.barrier()
    if rank == 0:
        single = dp.DeepPot(m, t, device=local)
        cs, vs = c.copy(), v.copy()
        rs = single.run_md(cs, vs, mc)
        nw = lambda a, b: float(np.max(np.abs(a - b)) / np.max(np.abs(b)))
        out = {
            "world": world, "atoms": c.n_atoms,
            "pe": [[a.pe, b.pe] for a, b in zip(rd.thermo, rs.thermo)],
            "ke": [[a.ke, b.ke] for a, b in zip(rd.thermo, rs.thermo)],
            "pressure": [[a.pressure, b.pressure] for a, b in zip(rd.thermo, rs.thermo)],
            "pos_normwise": nw(pos, cs.pos), "vel_normwise": nw(vel, vs),
            # per-atom forces are summed in the single-GPU order (global-id rows + pair halo), so
            # the whole trajectory is bitwise independent of the GPU count
            "pos_bitwise": bool(np.array_equal(pos, cs.pos)), "vel_bitwise": bool(np.array_equal(vel, vs)),
            "force_evals": [rd.force_evals, rs.force_evals],
            "counters": [[rd.counters.rows_forward, rd.counters.rows_backward, rd.counters.extrapolations],
                         [rs.counters.rows_forward, rs.counters.rows_backward, rs.counters.extrapolations]],
            "max_drift": [rd.max_drift_seen, rs.max_drift_seen],
        }
        path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/dist_md_check.json"
        Path(path).parent.mkdir(parents=True, exist_ok=True)
        Path(path).write_text(json.dumps(out, indent=1))
        print(json.dumps(out)[:2000])
    dist.barrier()
    pot.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
