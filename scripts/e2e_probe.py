"""Host-side breakdown of the public seed-supergraph path (C3 image)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1509_06004_b200 import LambdaSchedule, _native, synth, solve_seed_supergraph
from paper_1509_06004_b200.supergraph import check_seed_supergraph

imgs = int(sys.argv[1]) if len(sys.argv) > 1 else 1
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 5      # 1: the C2 single-seed supergraph
probs = []
for i in range(imgs):
    probs += synth.generate(500, 375, rows, rows, rng_seed=i, types=("A", "B") if rows > 1 else ("A",)).problems
sched = LambdaSchedule(synth.L20)
s = _native.solver_for_thread(0)
for rep in range(4):
    t0 = time.perf_counter(); check_seed_supergraph(probs, sched, "auto")
    t1 = time.perf_counter(); s.seed_stage(500, 375, probs, sched.values, "auto")
    t2 = time.perf_counter(); s.seed_run()
    t3 = time.perf_counter(); sw, fl, lab = s.seed_fetch(True)
    t4 = time.perf_counter(); res = solve_seed_supergraph(probs, sched, "auto", device=0)
    t5 = time.perf_counter()
    print(f"check {1e3*(t1-t0):.1f} stage {1e3*(t2-t1):.1f} run {1e3*(t3-t2):.1f} fetch {1e3*(t4-t3):.1f} "
          f"| public api {1e3*(t5-t4):.1f} ms (dev {s.stats()['ms_device']:.1f})")
