"""Domain decomposition host logic on CPU (no GPU): partition_domain parity with the reference,
ghost completeness (acceptance.cpp:388-417) and exchange-plan consistency across 2 gloo ranks."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle_lib as O
import paper_2201_01446_b200 as dp

needs_ref = pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built (no /root/reference)")


@needs_ref
@pytest.mark.parametrize("seed,w", [(871, 2), (872, 3), (873, 6)])
def test_partition_matches_reference(seed, w):
    import ctypes as C
    c = dp.make_random_config(24, 2, 10.0, 1.4, seed)
    owner, gm = dp.partition_domain(c, w, 4.5)
    n = c.n_atoms
    axis = C.c_int()
    ro = np.empty(n, dtype=np.int32)
    rg = np.empty((w, n), dtype=np.uint8)
    O._chk(O.ref().ref_partition_domain(n, dp._dp(c.pos), dp._dp(c.h), dp._u8(c.periodic), w, 4.5,
                                        C.byref(axis), dp._ip(ro), dp._u8(rg)), O.ref(), "ref_last_error")
    assert np.array_equal(owner, ro)
    assert np.array_equal(gm, rg.astype(bool))


@pytest.mark.parametrize("w", [2, 3, 4])
def test_ghost_audit_subset_lists_equal_global(w):
    """Every pair the global list knows is visible through owned + ghosts (same entries). The
    local order is owned-first, so a row's entry order can differ from the global row's; the
    entry sets (global id, shift) must be identical."""
    c = dp.gen_config("copper-like", 6, 5, 5, 0.1, 3)
    cutoff = 8.0 + 2.0
    glob = O.or_neighbor_list(c, cutoff)
    for r in range(w):
        plan = dp.dist_plan(c, w, r, cutoff)
        lg = plan["lgid"]
        sub = dp.AtomicConfig(c.pos[lg], c.type[lg], c.h, c.periodic)
        loc = O.or_neighbor_list(sub, cutoff)
        for k in np.nonzero(plan["center"])[0]:
            i = lg[k]
            gj, gs = glob.row(i)
            lj, ls = loc.row(k)
            a = sorted(zip(lg[lj].tolist(), map(tuple, ls.tolist())))
            b = sorted(zip(gj.tolist(), map(tuple, gs.tolist())))
            assert a == b, (r, i)


def _rank_main(rank, world, port, cfgd, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = dp.AtomicConfig(cfgd["pos"], cfgd["type"], cfgd["h"])
    plan = dp.dist_plan(c, world, rank, 10.0)
    mine = {p: plan["send"][p].tolist() for p in range(world)}
    theirs = [None] * world
    dist.all_gather_object(theirs, mine)
    owned = plan["lgid"][plan["center"]].tolist()
    all_owned = [None] * world
    dist.all_gather_object(all_owned, owned)
    ok = True
    for p in range(world):
        # what p sends to me must be exactly my ghosts owned by p, in the same order
        ok &= theirs[p][rank] == plan["recv"][p].tolist()
    flat = sorted(sum(all_owned, []))
    ok &= flat == list(range(c.n_atoms))
    ghosts = set(plan["lgid"][~plan["center"]].tolist())
    ok &= ghosts == set(sum((plan["recv"][p].tolist() for p in range(world)), []))
    q.put((rank, bool(ok), len(owned), len(ghosts)))
    dist.destroy_process_group()


def test_two_rank_exchange_plan_gloo():
    c = dp.gen_config("copper-like", 12, 5, 5, 0.1, 11)
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    cfgd = {"pos": c.pos, "type": c.type, "h": c.h}
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, cfgd, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _, _ in res), res
    assert sum(n for _, _, n, _ in res) == c.n_atoms
    assert all(g > 0 for _, _, _, g in res)
