"""Two handles evaluating concurrently on separate streams vs one (tools helper, not product)."""
import sys, threading, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2201_01446_b200 as dp
m = dp.gen_model("copper-like", 7); t = dp.build_tables(m, 0.01)
cells = int(sys.argv[1]) if len(sys.argv) > 1 else 20
c = dp.gen_config("copper-like", cells, cells, cells, 0.1, 11)
pots = [dp.DeepPot(m, t), dp.DeepPot(m, t)]
for p in pots:
    p.set_skin(2.0)
    for _ in range(3): p.compute(c)
K = 30
a = time.perf_counter()
for _ in range(K): pots[0].compute(c)
single = (time.perf_counter() - a) / K
def run(p):
    for _ in range(K): p.compute(c)
th = [threading.Thread(target=run, args=(p,)) for p in pots]
a = time.perf_counter()
for x in th: x.start()
for x in th: x.join()
dual = (time.perf_counter() - a) / K
print(f"atoms {c.n_atoms}: single {single*1e3:.2f} ms/eval, two concurrent {dual*1e3:.2f} ms per pair -> {2*single/dual:.2f}x throughput")
