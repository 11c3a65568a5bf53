"""Ad-hoc device probe: solve synthetic configs and print stats/timings.

    python scripts/probe.py [c1|c2|c3|c4] [--iters K] [--sweeps P] [--reps R]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1509_06004_b200 import LambdaSchedule, _native, synth  # noqa: E402
from paper_1509_06004_b200.parametric import DEFAULT_LAMBDA_VALUES  # noqa: E402

CFG = {
    "c1": dict(w=160, h=120, rows=1, cols=1, lams=DEFAULT_LAMBDA_VALUES, types=("A",)),
    "c2": dict(w=500, h=375, rows=1, cols=1, lams=synth.L20, types=("A",)),
    "c3": dict(w=500, h=375, rows=5, cols=5, lams=synth.L20, types=("A", "B")),
    "c4": dict(w=1920, h=1080, rows=1, cols=1, lams=synth.C4_LAMBDAS, types=("A",)),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg", nargs="?", default="c2")
    ap.add_argument("--iters", type=int, default=None)
    ap.add_argument("--sweeps", type=int, default=None)
    ap.add_argument("--chunk", type=int, default=None)
    ap.add_argument("--relabel", type=int, default=None)
    ap.add_argument("--persistent", type=int, default=None)
    ap.add_argument("--budget", type=int, default=None)
    ap.add_argument("--pbfs", type=int, default=None)
    ap.add_argument("--graph", type=int, default=None)
    ap.add_argument("--warp", type=int, default=None)
    ap.add_argument("--trace", action="store_true")
    ap.add_argument("--chain", type=int, default=None)
    ap.add_argument("--multi", type=int, default=None)
    ap.add_argument("--check", action="store_true", help="compare flows with a chain=1 solve")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--nprob", type=int, default=None, help="problems per device batch")
    ap.add_argument("--knob", action="append", default=[], help="name=value (any pmf_solver_set knob)")
    ap.add_argument("--images", type=int, default=1, help="images per device batch (rng_seed 0..)")
    ap.add_argument("--synth", action="store_true", help="planes derived on the device (pmf_synth_stage)")
    a = ap.parse_args()
    c = CFG[a.cfg]
    probs = []
    for i in range(a.images):
        b = synth.generate(c["w"], c["h"], c["rows"], c["cols"], rng_seed=i, types=c["types"])
        probs += b.problems
    probs = probs if a.nprob is None else probs[:a.nprob]
    s = _native.Solver(0)
    for kv in a.knob:
        kn, kv_ = kv.split("=")
        s.set(kn, int(kv_))
    if a.iters: s.set("push_iters", a.iters)
    if a.sweeps: s.set("push_sweeps", a.sweeps)
    if a.chunk: s.set("bfs_chunk", a.chunk)
    if a.relabel is not None: s.set("relabel_every", a.relabel)
    if a.persistent is not None: s.set("persistent", a.persistent)
    if a.budget is not None: s.set("push_budget", a.budget)
    if a.pbfs is not None: s.set("persistent_bfs", a.pbfs)
    if a.graph is not None: s.set("graph", a.graph)
    if a.warp is not None: s.set("warp", a.warp)
    if a.chain is not None: s.set("chain", a.chain)
    if a.multi is not None: s.set("bfs_multi", a.multi)
    ref = None
    if a.check:
        r0 = _native.Solver(0, chain=1)
        ref = r0.solve_seed_batch(c["w"], c["h"], probs, c["lams"], "auto")
        r0.close()
    devs = []
    for r in range(a.reps):
        t0 = time.perf_counter()
        if a.synth:
            from paper_1509_06004_b200.synth_device import generate_images
            ib = generate_images(c["w"], c["h"], c["rows"], c["cols"], range(a.images), c["types"])
            s.synth_stage(ib.images, ib.coords, ib.types, c["lams"], "auto")
        else:
            s.seed_stage(c["w"], c["h"], probs, c["lams"], "auto")
        t1 = time.perf_counter()
        s.seed_run()
        t2 = time.perf_counter()
        sw, flows, labels = s.seed_fetch(True)
        t3 = time.perf_counter()
        dt = t3 - t0
        st = s.stats()
        devs.append(st["ms_device"])
        cuts = flows.size
        if a.trace and r == a.reps - 1:
            tr = s.trace()
            print("trace push (us, tiles):", [(u, t) for k, u, t, _ in tr if k == 0])
            print("trace bfs  (us, tiles):", [(u, t) for k, u, t, _ in tr if k == 1][:30])
            print("timeline (kind, start_us, span_us, gap_us):")
            for i, (k, u, t, st0) in enumerate(tr):
                gap = st0 - (tr[i - 1][3] + tr[i - 1][1]) if i else 0.0
                print(f"  {k} {st0:9.1f} {u:8.1f} {gap:7.1f} tiles={t}")
        if st.get("async_mode") and r == a.reps - 1:
            print("busy ms (CTA-summed):", s.busy(), "kernel ms", round(st["ms_async"], 3))
        if ref is not None:
            import numpy as np
            ok = bool((ref[1] == flows).all()) and bool(np.array_equal(ref[2], labels))
            print("check vs chain=1:", "OK" if ok else "MISMATCH")
        keep = ("cycles", "push_tile_passes", "bfs_tile_passes", "label_tile_passes", "push_sweeps",
                "bfs_sweeps", "ms_device", "ms_push", "ms_bfs", "ms_labels", "launches", "graph_builds",
                "steps", "grids", "scan_tile_passes", "ms_async")
        print(json.dumps(dict(cfg=a.cfg, args=" ".join(sys.argv[2:]), rep=r,
                              wall_ms=round(dt * 1e3, 2), stage_ms=round((t1 - t0) * 1e3, 2),
                              run_ms=round((t2 - t1) * 1e3, 2), fetch_ms=round((t3 - t2) * 1e3, 2),
                              cuts_per_s=round(cuts / dt, 1),
                              flow=int(flows.sum()),
                              med_dev_ms=round(sorted(devs[1:] or devs)[len(devs[1:] or devs) // 2], 3),
                              **{k: (round(st[k], 3) if isinstance(st[k], float) else st[k]) for k in keep})))


if __name__ == "__main__":
    main()
