"""One small solve for compute-sanitizer runs (scripts/sanitize.sh).

    python scripts/sanitize_case.py c1-async | c1-sync | c3-async | comp | wide

c1-async  C1 seed supergraph through k_async (persistent queue kernel)
c1-sync   C1 through the step-synchronous engine (k_push, k_bfs_sink /
          k_wbfs_*, cooperative multi-sweep BFS, graph-driven loop)
c3-async  one C3 CPMC image (50 warm-start chains) through k_async
comp      a composite with a swapped span (k_load_comp path + certificate)
*-host    the same case with the host-driven loop (graph=0)
wide      the int64 state variant on a CAP_MAX-heavy graph
synth     a synthetic image batch, planes built on the device (async; -sync: step mode)
stream    the batch stream: runs launched behind each other on three solvers
Each case checks its result against the oracle, so a sanitizer run that
perturbs scheduling still has to produce the reference's cuts.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1509_06004_b200 import (CAP_MAX, GridGraph, LambdaSchedule, _native, admit, apply_swap,  # noqa: E402
                                   join, maxflow_pushrelabel, solve_composite, solve_seed_supergraph,
                                   synth)


def check_seed(probs, sched, res, k=3):
    for pi in range(min(k, len(probs))):
        p = probs[pi]
        for li in (0, len(sched) // 2, len(sched) - 1):
            src, snk, nbr = oracle.instantiate(p.unary_base, p.unary_slope, p.sink_base, p.pairwise,
                                               p.fg_seeds, p.bg_seeds, sched[li])
            f, lab, _ = oracle.solve(p.width, p.height, src, snk, nbr)
            c = res.cuts[pi * len(sched) + li]
            assert c.flow == f and np.array_equal(c.labels, lab), (pi, li)


def main(case):
    s = _native.solver_for_thread(0)
    if case.endswith("-host"):
        # host-driven loop (knob graph=0): racecheck cannot run the solve
        # graph's conditional nodes, so the step-synchronous kernels are
        # checked through the host loop (same kernels)
        s.set("graph", 0)
        case = case[:-5]
    if case in ("c1-async", "c1-sync"):
        s.set("async", 1 if case == "c1-async" else 0)
        b = synth.generate(160, 120, 1, 1, rng_seed=0)
        sched = LambdaSchedule.default()
        res = solve_seed_supergraph(b.problems, sched, "auto")
        assert res.flow == 27814225
        check_seed(b.problems, sched, res)
    elif case == "c3-async":
        s.set("async", 1)
        b = synth.generate(500, 375, 5, 5, rng_seed=0, types=("A", "B"))
        sched = LambdaSchedule(synth.L20)
        res = solve_seed_supergraph(b.problems, sched, "auto")
        check_seed(b.problems, sched, res, k=1)
    elif case == "comp":
        b = synth.generate(96, 72, 1, 1, rng_seed=1)
        from paper_1509_06004_b200 import instantiate
        g1, g2 = instantiate(b.problems[0], 3), instantiate(b.problems[0], 40)
        comp, lay = join([apply_swap(g1), g2], swapped=[True, False])
        cut = solve_composite(comp, lay)
        f, lab, _ = oracle.solve(comp.width, comp.height, comp.src_cap, comp.snk_cap, comp.nbr_cap,
                                 [(x.offset, x.width, x.swapped) for x in lay.segments])
        assert cut.flow == f and np.array_equal(cut.labels, lab)
    elif case == "wide":
        rng = np.random.default_rng(7)
        w, h = 40, 30
        nb = rng.choice([0, 5, CAP_MAX], (4, h, w))
        nb[0][:, 0] = nb[1][:, -1] = 0
        nb[2][0, :] = nb[3][-1, :] = 0
        g = admit(GridGraph(w, h, rng.choice([0, 9, CAP_MAX], w * h), rng.choice([0, 7, CAP_MAX], w * h),
                            nb.reshape(4, -1)))
        cut = maxflow_pushrelabel(g)
        assert s.stats()["wide_mode"] == 1
        f, lab, _ = oracle.solve(w, h, g.src_cap, g.snk_cap, g.nbr_cap)
        assert cut.flow == f and np.array_equal(cut.labels, lab)
    elif case in ("synth", "synth-sync"):
        # on-device synthesis: k_synth_planes (ragged 53x37 images: the
        # scalar store path) and k_synth_pw at the start of the run
        from paper_1509_06004_b200.synth_device import generate_images, solve_image_batch
        s.set("async", 1 if case == "synth" else 0)
        b = generate_images(53, 37, 1, 2, rng_seeds=(4, 5), types=("A", "B"))
        sched = LambdaSchedule(synth.L20[:6])
        res = solve_image_batch(b, sched)
        check_seed(b.problems(), sched, res, k=4)
    elif case == "stream":
        # batch stream: three solvers, each run launched behind the previous
        # one (pmf_seed_launch with `after`), an image batch in the middle
        from paper_1509_06004_b200 import solve_seed_supergraphs
        from paper_1509_06004_b200.synth_device import generate_images
        sched = LambdaSchedule(synth.L20[:6])
        p0 = synth.generate(96, 64, 1, 2, rng_seed=1, types=("A", "B")).problems
        b1 = generate_images(96, 64, 1, 2, rng_seeds=(2,), types=("A", "B"))
        p2 = synth.generate(96, 64, 1, 2, rng_seed=3, types=("A", "B")).problems
        for probs, res in zip((p0, b1.problems(), p2), solve_seed_supergraphs([p0, b1, p2], sched)):
            check_seed(probs, sched, res, k=4)
    else:
        raise SystemExit(f"unknown case {case}")
    print(case, "ok")


if __name__ == "__main__":
    main(sys.argv[1])
