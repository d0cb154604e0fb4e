"""Quick GPU parity probe used during development (not part of the test suite)."""
import sys, time, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2201_01446_b200 as dp
import oracle_lib as O

def nw(a, b):
    return O.normwise(a, b)

m = dp.gen_model("copper-like", 7)
tb = dp.build_tables(m, 0.01)
c = dp.gen_config("copper-like", 8, 8, 8, 0.1, 11)
pot = dp.DeepPot(m, tb)
for cut in (8.0, 10.0):
    t0 = time.time(); lg = pot.neighbor_list(c, cut); t1 = time.time()
    lo = O.or_neighbor_list(c, cut)
    print("nlist", cut, "equal", O.lists_equal(lg, lo), lg.j.size, lo.j.size, "%.3fs" % (t1 - t0), flush=True)
ro, co = O.or_compute(c, m, tb)
for skin in (0.0, 2.0):
    pot.set_skin(skin)
    t0 = time.time(); r = pot.compute(c); t1 = time.time()
    print("skin", skin, "E gpu %.17g oracle %.17g rel %.3e" % (r.energy, ro.energy, abs(r.energy - ro.energy) / abs(ro.energy)),
          "F %.3e V %.3e Ei %.3e" % (nw(r.forces, ro.forces), nw(r.virial, ro.virial), nw(r.per_atom_energy, ro.per_atom_energy)),
          pot.counters, co, "%.3fs" % (t1 - t0), flush=True)
# small multi-type multi-image
mt = dp.make_test_model(2, 6, 8, 20, 2, [18, 18], 6.0, 5.0, 401)
tt = dp.build_tables(mt, 0.05)
for trial in range(3):
    cf = dp.make_random_config(10, 2, 9.0, 1.8, 500 + trial)
    p2 = dp.DeepPot(mt, tt)
    r = p2.compute(cf)
    ro, co = O.or_compute(cf, mt, tt)
    print("small", trial, "E rel %.3e F %.3e V %.3e" % (abs(r.energy - ro.energy) / abs(ro.energy), nw(r.forces, ro.forces), nw(r.virial, ro.virial)), p2.counters, co)
    lg = p2.neighbor_list(cf, 7.0); lo = O.or_neighbor_list(cf, 7.0)
    print("  nlist multi-image equal", O.lists_equal(lg, lo), lg.j.size)
# timing 32k
c2 = dp.gen_config("copper-like", 20, 20, 20, 0.1, 11)
pot.set_skin(2.0)
r = pot.compute(c2)
import ctypes
t0 = time.time()
for _ in range(5): r = pot.compute(c2)
t1 = time.time()
print("C2 compute x5 %.3f s/eval, E %.17g (golden -5040.6583216965946)" % ((t1 - t0) / 5, r.energy))
