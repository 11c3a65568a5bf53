"""Batch-stream timeline: per batch the device time of its run and the wall
time between consecutive results (solve_seed_supergraphs).

    python scripts/stream_probe.py [images_per_batch] [batches]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1509_06004_b200 import LambdaSchedule, _native, solve_seed_supergraphs, synth  # noqa: E402
from paper_1509_06004_b200 import supergraph as sg  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 1
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 8
sched = LambdaSchedule(synth.L20)


def batch(b):
    out = []
    for i in range(k):
        out += synth.generate(500, 375, 5, 5, rng_seed=b * k + i, types=("A", "B")).problems
    return out


for rep in range(2):
    bs = [batch(b + 10 * rep) for b in range(nb)]
    sv = _native.pipeline_solvers(0, 3)
    marks = []
    orig_wait = _native.Solver.seed_wait

    def wait(self, _o=orig_wait):
        t = time.perf_counter()
        _o(self)
        marks.append((t, time.perf_counter(), self.stats()["ms_device"]))
    _native.Solver.seed_wait = wait
    t0 = time.perf_counter()
    ys = []
    for r in solve_seed_supergraphs(bs, sched):
        ys.append(time.perf_counter())
        del r
    T = time.perf_counter() - t0
    _native.Solver.seed_wait = orig_wait
    dev = sum(m[2] for m in marks)
    print(f"rep {rep}: {nb} batches x {k} images: wall {1e3 * T:.1f} ms, device sum {dev:.1f} ms, "
          f"per image wall {1e3 * T / nb / k:.2f} dev {dev / nb / k:.2f}")
    print("  wait blocked ms:", [round(1e3 * (b - a), 1) for a, b, _ in marks])
    print("  device ms:", [round(d, 1) for _, _, d in marks])
    print("  gaps between results ms:", [round(1e3 * (b - a), 1) for a, b in zip([t0] + ys, ys)])
