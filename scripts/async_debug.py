"""Compare asynchronous vs step-synchronous solves of a C3 batch."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1509_06004_b200 import _native, synth

imgs = int(sys.argv[1]) if len(sys.argv) > 1 else 8
knobs = dict(kv.split("=") for kv in sys.argv[2:])
knobs = {k: int(v) for k, v in knobs.items()}
probs = []
for i in range(imgs):
    probs += synth.generate(500, 375, 5, 5, rng_seed=i, types=("A", "B")).problems
ref = _native.Solver(0, **{"async": 0})
sw, fr, lr = ref.solve_seed_batch(500, 375, probs, synth.L20, "auto")
print("swapped problems:", int(sw.sum()))
for rep in range(3):
    s = _native.Solver(0, verify=0, **knobs)
    s.seed_stage(500, 375, probs, synth.L20, "auto")
    try:
        s.seed_run()
    except Exception as e:
        print("run error:", e)
    _, fa, la = s.seed_fetch(True)
    print("stats", {k: s.stats()[k] for k in ("cycles", "steps", "push_tile_passes", "bfs_tile_passes")})
    bad = np.argwhere(fa != fr)
    badl = np.argwhere((la != lr).any(axis=2))
    print(f"{knobs} rep {rep}: flow mismatches {len(bad)}, label mismatches {len(badl)}", bad[:10].tolist(),
          [(int(p), int(l), bool(sw[p]), int(fa[p, l] - fr[p, l])) for p, l in bad[:10]])
    s.close()
