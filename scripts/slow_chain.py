"""Phase durations of one chain of a C3 image: in the batch vs alone."""
import os, sys, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1509_06004_b200 import _native, synth
g = int(sys.argv[1]) if len(sys.argv) > 1 else 34
p = synth.generate(500, 375, 5, 5, rng_seed=0, types=("A", "B")).problems

def summary(s, grid):
    ph = s.phases(grid)
    tot = collections.defaultdict(float); cnt = collections.Counter()
    for i in range(len(ph) - 1):
        tot[ph[i][0]] += ph[i + 1][1] - ph[i][1]
        cnt[ph[i][0]] += 1
    return {k: (cnt[k], round(tot[k] / 1e3, 2)) for k in tot}, round(ph[-1][1] / 1e3, 2)

s = _native.Solver(0, phase_log=1)
for r in range(2):
    s.solve_seed_batch(500, 375, p, synth.L20, "auto")
print("batch: phases (count, ms)", *summary(s, g))
s2 = _native.Solver(0, phase_log=1, chain=20)
for r in range(2):
    s2.solve_seed_batch(500, 375, [p[g]], synth.L20, "auto")
print("alone: phases (count, ms)", *summary(s2, 0))
