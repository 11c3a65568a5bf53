"""Several solvers sharing one GPU (one host thread and stream each, 1/L of
the resident CTAs each), C3 problems split across them."""
import os, sys, time, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1509_06004_b200 import _native, synth

lanes = int(sys.argv[1]); imgs = int(sys.argv[2]) if len(sys.argv) > 2 else 1
pbfs = int(sys.argv[3]) if len(sys.argv) > 3 else 1
probs = []
for i in range(imgs):
    probs += synth.generate(500, 375, 5, 5, rng_seed=i, types=("A", "B")).problems
parts = [probs[i::lanes] for i in range(lanes)]
sv = [_native.Solver(0, grid_div=lanes, persistent_bfs=pbfs) for _ in range(lanes)]
for s, p in zip(sv, parts):
    s.seed_stage(500, 375, p, synth.L20, "auto")
res = [None] * lanes
def work(i):
    sv[i].seed_run()
for rep in range(4):
    t0 = time.perf_counter()
    th = [threading.Thread(target=work, args=(i,)) for i in range(lanes)]
    [t.start() for t in th]; [t.join() for t in th]
    dt = time.perf_counter() - t0
    flows = sum(int(s.seed_fetch(False)[1].sum()) for s in sv)
    print(f"lanes {lanes} imgs {imgs} pbfs {pbfs}: {1e3*dt:.1f} ms  ({1e3*dt/imgs:.1f} ms/img) flow {flows} dev {[round(s.stats()['ms_device'],1) for s in sv]}")
