"""Stress: a long batch stream mixing asynchronous (1-2 image) and
step-synchronous (8 image) batches, host-staged and device-synthesised,
overlap on; every result compared with the single call of the same batch.

    python scripts/stress_stream.py [batches]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1509_06004_b200 import LambdaSchedule, solve_seed_supergraph, solve_seed_supergraphs, synth  # noqa: E402
from paper_1509_06004_b200.synth_device import generate_images  # noqa: E402

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 24
sched = LambdaSchedule(synth.L20)
rng = np.random.default_rng(5)
batches = []
for b in range(nb):
    k = int(rng.choice([1, 1, 2, 8]))
    seeds = [int(s) for s in rng.integers(0, 256, k)]
    if rng.random() < 0.5:
        batches.append(generate_images(500, 375, 5, 5, seeds, ("A", "B")))
    else:
        probs = []
        for s in seeds:
            probs += synth.generate(500, 375, 5, 5, rng_seed=s, types=("A", "B")).problems
        batches.append(probs)
bad = 0
for b, res in zip(batches, solve_seed_supergraphs(batches, sched)):
    probs = b.problems() if hasattr(b, "problems") and callable(b.problems) else b
    want = solve_seed_supergraph(probs, sched)
    ok = ([c.flow for c in res.cuts] == [c.flow for c in want.cuts] and
          all(np.array_equal(x.labels, y.labels) for x, y in zip(res.cuts, want.cuts)))
    bad += not ok
print(f"stress: {nb} batches, {bad} mismatches")
sys.exit(1 if bad else 0)
