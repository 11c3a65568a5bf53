"""Batch-stream timeline: when each batch was staged, launched, waited for
and fetched (solve_seed_supergraphs), relative to the stream start.

    python scripts/stream_probe.py [images_per_batch] [batches] [synth]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1509_06004_b200 import LambdaSchedule, _native, solve_seed_supergraphs, synth  # noqa: E402
from paper_1509_06004_b200.synth_device import generate_images  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 1
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 8
use_synth = len(sys.argv) > 3 and sys.argv[3] == "synth"
sched = LambdaSchedule(synth.L20)


def batch(b):
    if use_synth:
        return generate_images(500, 375, 5, 5, [b * k + i for i in range(k)], ("A", "B"))
    out = []
    for i in range(k):
        out += synth.generate(500, 375, 5, 5, rng_seed=b * k + i, types=("A", "B")).problems
    return out


for kv in filter(None, os.environ.get("KNOBS", "").split(",")):   # e.g. KNOBS=async=1
    k_, v_ = kv.split("=")
    _native.configure(**{k_: int(v_)})
log = []
for name in ("seed_stage", "synth_stage", "seed_launch", "seed_wait", "seed_fetch") if os.environ.get("TRACE") else ():
    orig = getattr(_native.Solver, name)

    def wrap(self, *a, _o=orig, _n=name, **kw):
        t = time.perf_counter()
        r = _o(self, *a, **kw)
        log.append((_n, id(self) % 1000, t, time.perf_counter()))
        return r
    setattr(_native.Solver, name, wrap)

if os.environ.get("TRACE"):
    from paper_1509_06004_b200 import supergraph as _sg
    for name in ("check_seed_supergraph", "_layout_skeleton", "_collect"):
        orig = getattr(_sg, name)

        def wrap2(*a, _o=orig, _n=name, **kw):
            t = time.perf_counter()
            r = _o(*a, **kw)
            log.append((_n, 0, t, time.perf_counter()))
            return r
        setattr(_sg, name, wrap2)

for rep in range(2):
    bs = [batch(b + 10 * rep) for b in range(nb)]
    log.clear()
    t0 = time.perf_counter()
    ys = []
    for r in solve_seed_supergraphs(bs, sched, overlap_us=int(os.environ.get("OVERLAP", 20))):
        ys.append(time.perf_counter())
        del r
    T = time.perf_counter() - t0
    print(f"rep {rep}: {nb} batches x {k} images{' (synth)' if use_synth else ''}: wall {1e3 * T:.1f} ms, "
          f"{1e3 * T / nb / k:.2f} ms/image")
    for n, sid, a, b in sorted(log, key=lambda e: e[2]):
        print(f"  {n:12s} solver {sid:3d} {1e3 * (a - t0):8.1f} -> {1e3 * (b - t0):8.1f}  ({1e3 * (b - a):7.1f} ms)")
    print("  results at", [round(1e3 * (y - t0), 1) for y in ys])

# device-resident time of the same batches (stage untimed, run timed on the device)
s = _native.solver_for_thread(0)
dev = 0.0
for b in bs:
    if use_synth:
        s.synth_stage(b.images, b.coords, b.types, sched.values, "auto")
    else:
        s.seed_stage(500, 375, b, sched.values, "auto")
    s.seed_run()
    dev += s.stats()["ms_device"]
print(f"device-resident: {dev:.1f} ms, {dev / nb / k:.2f} ms/image (stream wall above)")
