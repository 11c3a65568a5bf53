"""Phase timeline of one lambda-graph of C2 (async solver, phase_log=1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1509_06004_b200 import _native, synth
p = synth.generate(500, 375, 1, 1, rng_seed=0).problems
lams = list(synth.L20) if len(sys.argv) < 2 or sys.argv[1] == "all" else [int(x) for x in sys.argv[1].split(",")]
s = _native.Solver(0, phase_log=1)
for r in range(3):
    s.solve_seed_batch(500, 375, p, lams, "auto")
print("device ms", round(s.stats()["ms_device"], 3), "lambdas", lams)
for g in range(len(lams)):
    ph = s.phases(g)
    if lams[g] in (3, 4, 5, 9) or len(lams) == 1:
        segs = [(ph[i][0], round(ph[i + 1][1] - ph[i][1], 1)) for i in range(len(ph) - 1)]
        print("lambda", lams[g], "end", ph[-1][1], segs)
