"""Device time of C2 lambda subsets solved together (cold grids)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1509_06004_b200 import _native, synth
p = synth.generate(500, 375, 1, 1, rng_seed=0).problems
s = _native.Solver(0)
sets = {"all20": list(synth.L20), "lam4": [4], "hard4": [3, 4, 5, 9], "hard6": [2, 3, 4, 5, 7, 9],
        "easy14": list(synth.L20[6:]), "lam4x2": None}
for name, lams in sets.items():
    if lams is None:
        continue
    ts = []
    for r in range(4):
        s.solve_seed_batch(500, 375, p, lams, "auto")
        ts.append(s.stats()["ms_device"])
    print(name, [round(t, 3) for t in ts])
