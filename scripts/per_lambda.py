"""Device time of each lambda-graph of a config solved alone (one grid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1509_06004_b200 import _native, synth
W, H = (500, 375) if len(sys.argv) < 2 else map(int, sys.argv[1].split("x"))
p = synth.generate(W, H, 1, 1, rng_seed=0).problems
s = _native.Solver(0)
out = []
for lam in synth.L20:
    ts = []
    for r in range(3):
        s.solve_seed_batch(W, H, p, [lam], "auto")
        st = s.stats()
        ts.append(st["ms_device"])
    out.append((lam, round(min(ts), 3), st["cycles"], st["push_tile_passes"], st["bfs_tile_passes"]))
for o in out:
    print("lambda %4d  ms %.3f  cycles %d  push %d  bfs %d" % o)
