"""Host-side phases of one public-API C5 batch (fresh CPMC images):
admission checks, stage (narrow + H2D), device run, fetch (D2H + unpack),
CutResult construction.  Prints ms per phase (median over fresh batches).

    python scripts/e2e_phases.py [images]
"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1509_06004_b200 import LambdaSchedule, _native, solve_seed_supergraph, synth  # noqa: E402
from paper_1509_06004_b200.grid import CutResult  # noqa: E402
from paper_1509_06004_b200.supergraph import check_seed_supergraph  # noqa: E402

imgs = int(sys.argv[1]) if len(sys.argv) > 1 else 8
sched = LambdaSchedule(synth.L20)
s = _native.solver_for_thread(0)
rows = []
for rep in range(5):
    probs = []
    for i in range(imgs):
        probs += synth.generate(500, 375, 5, 5, rng_seed=100 + rep * imgs + i, types=("A", "B")).problems
    t = [time.perf_counter()]
    check_seed_supergraph(probs, sched, "auto")
    t.append(time.perf_counter())
    s.seed_stage(500, 375, probs, sched.values, "auto")
    t.append(time.perf_counter())
    s.seed_run()
    t.append(time.perf_counter())
    sw, fl, lab = s.seed_fetch(True)
    t.append(time.perf_counter())
    flat = fl.reshape(-1)
    cuts = [CutResult._trusted(int(f), l) for f, l in zip(flat, lab.reshape(flat.size, -1))]
    t.append(time.perf_counter())
    del cuts, lab
    probs2 = []
    for i in range(imgs):
        probs2 += synth.generate(500, 375, 5, 5, rng_seed=200 + rep * imgs + i, types=("A", "B")).problems
    t0 = time.perf_counter()
    res = solve_seed_supergraph(probs2, sched, "auto")
    t1 = time.perf_counter()
    del res
    rows.append([1e3 * (b - a) for a, b in zip(t, t[1:])] + [1e3 * (t1 - t0), s.stats()["ms_device"]])
names = ("check", "stage", "run", "fetch", "results", "api_total", "device")
med = [statistics.median(r[k] for r in rows[2:]) for k in range(len(names))]
print({n: round(v, 1) for n, v in zip(names, med)}, "ms per", imgs, "images")
pl = [np.arange(187500, dtype=np.int64) % 64 for _ in range(600)]
for _ in range(3):
    t = time.perf_counter()
    _native.plane_stats(pl)
    a = time.perf_counter() - t
    t = time.perf_counter()
    [(x.min(), x.max(), x.sum()) for x in pl]
    b = time.perf_counter() - t
print(f"plane stats 600 planes: native {1e3 * a:.1f} ms, numpy {1e3 * b:.1f} ms")
