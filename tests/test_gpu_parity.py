"""Parity of the CUDA engine against the reference (golden vectors) and the
CPU oracle.  Integer capacities: flows and label masks must be bit-exact."""

import os

import numpy as np
import pytest

import oracle
from conftest import (GOLDEN, load_composites, load_kat, load_random, load_seed_supergraphs,
                      load_synth)
from paper_1509_06004_b200 import (CAP_MAX, GridGraph, LambdaSchedule, SeedProblem, admit,
                                   apply_swap, build_seed_supergraph, cut_cost, join,
                                   maxflow_many, maxflow_pushrelabel, solve_composite,
                                   solve_composites, solve_schedule_sequential,
                                   solve_seed_supergraph, split, synth)

pytestmark = pytest.mark.gpu


def grid(w, h, s, t, nb):
    return admit(GridGraph(w, h, np.asarray(s), np.asarray(t), np.asarray(nb)))


def test_kat_fixtures(engine):
    for name, k in load_kat().items():
        r = maxflow_pushrelabel(grid(k["width"], k["height"], k["src"], k["snk"], k["nbr"]))
        assert r.flow == k["flow"], name
        assert r.labels.tolist() == k["labels"], name


@pytest.mark.parametrize("name", ["random_8x8_seed101.npz", "random_3x3_seed102.npz"])
def test_random_sweeps_one_batch(engine, name):
    """test_acceptance.py:34-60 fixtures, all graphs in ONE device batch."""
    cases = load_random(name)
    got = maxflow_many([grid(w, h, s, t, nb) for (w, h, s, t, nb, _, _) in cases])
    for r, (*_, flow, labels) in zip(got, cases):
        assert r.flow == flow
        assert np.array_equal(r.labels, labels)


def test_random_sweep_individually(engine):
    for (w, h, s, t, nb, flow, labels) in load_random("random_8x8_seed101.npz")[:60]:
        r = maxflow_pushrelabel(grid(w, h, s, t, nb))
        assert r.flow == flow and np.array_equal(r.labels, labels)


def test_composites_with_swapped_spans(engine):
    """Composite-level labels incl. swapped spans and padded rows
    (supergraph.py:201-206)."""
    from paper_1509_06004_b200 import Segment, SupergraphLayout
    cases = load_composites()
    tasks = []
    for (w, h, s, t, nb, rec) in cases:
        segs = tuple(Segment(i, o, sw_w, bool(f)) for i, (o, sw_w, f) in enumerate(rec["segments"]))
        tasks.append((grid(w, h, s, t, nb), SupergraphLayout(segs, (), h)))
    got = solve_composites(tasks)
    for r, (*_, rec) in zip(got, cases):
        assert r.flow == rec["flow"]
        assert r.labels.tolist() == rec["labels"]
    # and one at a time through the drop-in entry point
    for (g, lay), (*_, rec) in list(zip(tasks, cases))[:10]:
        r = solve_composite(g, lay)
        assert r.flow == rec["flow"] and r.labels.tolist() == rec["labels"]


def _problems(case):
    W, H = case["width"], case["height"]
    return [SeedProblem(W, H, p["base"], p["slope"], p["sink"], p["pairwise"],
                        frozenset(p["fg"]), frozenset(p["bg"])) for p in case["problems"]]


def test_seed_supergraph_device_builder(engine):
    for case in load_seed_supergraphs():
        probs = _problems(case)
        res = solve_seed_supergraph(probs, LambdaSchedule(case["lambdas"]), case["mode"])
        assert [s.swapped for s in res.layout.segments] == case["swapped"]
        assert res.layout.total_width == case["composite_width"]
        assert [c.flow for c in res.cuts] == case["flows"]
        assert [c.labels.tolist() for c in res.cuts] == case["labels"]


def test_seed_supergraph_host_composite_path(engine):
    for case in load_seed_supergraphs():
        probs = _problems(case)
        comp, layout, originals = build_seed_supergraph(probs, LambdaSchedule(case["lambdas"]),
                                                        case["mode"])
        cut = solve_composite(comp, layout)
        assert cut.flow == case["composite_flow"]
        assert cut.labels.tolist() == case["composite_labels"]
        parts = split(layout, cut, originals)
        assert [p.flow for p in parts] == case["flows"]


def test_c1_supergraph(engine):
    """C1: 160x120, 1 seed, DEFAULT 20-lambda ladder, one supergraph."""
    g = load_synth("c1_160x120.npz")
    probs = synth.generate(160, 120, rng_seed=0).problems
    sched = LambdaSchedule(g["lambdas"])
    res = solve_seed_supergraph(probs, sched, "auto")
    assert res.flow == 27814225
    for j, (c, flow, lab) in enumerate(zip(res.cuts, g["flows"], g["labels"])):
        assert c.flow == flow, j
        assert np.array_equal(c.labels, lab), (j, int((c.labels != lab).sum()))
    comp, layout, originals = build_seed_supergraph(probs, sched, "auto")
    cut = solve_composite(comp, layout)
    assert cut.flow == 27814225
    parts = split(layout, cut, originals)
    for j, (p, flow, lab) in enumerate(zip(parts, g["flows"], g["labels"])):
        assert p.flow == flow, ("composite", j, p.flow, flow)
        assert np.array_equal(p.labels, lab), ("composite", j, int((p.labels != lab).sum()))


def test_c1_swapped_family_matches(engine):
    """Forcing the s-t swap must not change any decoded cut."""
    g = load_synth("c1_160x120.npz")
    probs = synth.generate(160, 120, rng_seed=0).problems
    res = solve_seed_supergraph(probs, LambdaSchedule(g["lambdas"]), "on")
    assert all(s.swapped for s in res.layout.segments)
    for c, flow, lab in zip(res.cuts, g["flows"], g["labels"]):
        assert c.flow == flow and np.array_equal(c.labels, lab)


@pytest.mark.skipif(not os.path.exists(os.path.join(GOLDEN, "c2_500x375.npz")),
                    reason="C2 fixture not generated")
def test_c2_sequential_and_supergraph(engine):
    """C2: 500x375, L20 ladder: per-lambda reference cuts."""
    g = load_synth("c2_500x375.npz")
    p = synth.generate(500, 375, rng_seed=0).problems[0]
    sched = LambdaSchedule(g["lambdas"])
    res = solve_seed_supergraph([p], sched, "auto")
    assert res.flow == 90475333
    for c, flow, lab in zip(res.cuts, g["flows"], g["labels"]):
        assert c.flow == flow and np.array_equal(c.labels, lab)
    seq = solve_schedule_sequential(p, sched)
    assert [c.flow for c in seq.cuts] == g["flows"]


def test_repeated_runs_bit_identical(engine):
    probs = synth.generate(160, 120, rng_seed=3).problems
    sched = LambdaSchedule.default()
    a = solve_seed_supergraph(probs, sched)
    b = solve_seed_supergraph(probs, sched)
    assert [c.flow for c in a.cuts] == [c.flow for c in b.cuts]
    assert all(x.labels.tobytes() == y.labels.tobytes() for x, y in zip(a.cuts, b.cuts))


def test_edge_shapes_vs_oracle(engine):
    """1xN, Nx1, tiles straddling 32-px boundaries, CAP_MAX seeds."""
    rng = np.random.default_rng(5)
    graphs = []
    for (w, h) in [(1, 1), (1, 40), (40, 1), (31, 33), (33, 31), (64, 64), (65, 3), (3, 97)]:
        n = w * h
        nb = rng.integers(0, 12, (4, h, w))
        nb[0][:, 0] = 0
        nb[1][:, -1] = 0
        nb[2][0, :] = 0
        nb[3][-1, :] = 0
        src = rng.integers(0, 15, n)
        snk = rng.integers(0, 15, n)
        src[rng.integers(0, n)] = CAP_MAX
        graphs.append(grid(w, h, src, snk, nb.reshape(4, -1)))
    got = maxflow_many(graphs)
    for g, r in zip(graphs, got):
        f, lab, _ = oracle.solve(g.width, g.height, g.src_cap, g.snk_cap, g.nbr_cap)
        assert r.flow == f and np.array_equal(r.labels, lab)
        assert cut_cost(g, r.labels) == r.flow


def test_wide_capacities_int32_edges(engine):
    """Arc pairs above 255 select the int32 residual layout."""
    rng = np.random.default_rng(9)
    graphs = []
    for _ in range(20):
        w, h = int(rng.integers(2, 40)), int(rng.integers(2, 40))
        n = w * h
        nb = rng.integers(0, 5000, (4, h, w))
        nb[0][:, 0] = 0
        nb[1][:, -1] = 0
        nb[2][0, :] = 0
        nb[3][-1, :] = 0
        graphs.append(grid(w, h, rng.integers(0, 20000, n), rng.integers(0, 20000, n),
                           nb.reshape(4, -1)))
    got = maxflow_many(graphs)
    for g, r in zip(graphs, got):
        f, lab, _ = oracle.solve(g.width, g.height, g.src_cap, g.snk_cap, g.nbr_cap)
        assert r.flow == f and np.array_equal(r.labels, lab)


def test_random_composites_vs_oracle(engine):
    rng = np.random.default_rng(77)
    tasks, ref = [], []
    for _ in range(12):
        k = int(rng.integers(1, 5))
        h = int(rng.integers(5, 45))
        graphs = []
        for _ in range(k):
            w = int(rng.integers(5, 45))
            nb = rng.integers(0, 30, (4, h, w))
            nb[0][:, 0] = 0
            nb[1][:, -1] = 0
            nb[2][0, :] = 0
            nb[3][-1, :] = 0
            graphs.append(grid(w, h, rng.integers(0, 60, w * h), rng.integers(0, 60, w * h),
                               nb.reshape(4, -1)))
        flags = [bool(rng.integers(0, 2)) for _ in graphs]
        comp, lay = join([apply_swap(g) if f else g for g, f in zip(graphs, flags)], swapped=flags)
        tasks.append((comp, lay))
        ref.append(oracle.solve(comp.width, comp.height, comp.src_cap, comp.snk_cap, comp.nbr_cap,
                                [(s.offset, s.width, s.swapped) for s in lay.segments]))
    for r, (f, lab, _) in zip(solve_composites(tasks), ref):
        assert r.flow == f and np.array_equal(r.labels, lab)


@pytest.mark.parametrize("i32", [False, True])
@pytest.mark.parametrize("plane,where", [("src", 0), ("snk", -1), ("nbr", 0), ("nbr", -1)])
def test_composite_staging_range_errors_leave_solver_usable(engine, i32, plane, where):
    """pmf_solve_composites(_i32) narrows and uploads the planes in pieces
    (src, snk, four neighbour quarters); a value outside [0, CAP_MAX] in any
    piece -- first or last composite, first or last plane -- is the
    reference's CapacityOverflowError, and the same solver then solves a valid
    request bit-exactly (oracle)."""
    from paper_1509_06004_b200 import CapacityOverflowError
    rng = np.random.default_rng(5)
    items = []
    for k in range(3):
        w, h = int(rng.integers(3, 40)), int(rng.integers(3, 40))
        nb = rng.integers(0, 25, (4, h, w))
        nb[0][:, 0] = 0
        nb[1][:, -1] = 0
        nb[2][0, :] = 0
        nb[3][-1, :] = 0
        items.append([w, h, rng.integers(0, 50, w * h), rng.integers(0, 50, w * h), nb.reshape(4, -1), None])
    bad = [list(it) for it in items]
    idx = {"src": 2, "snk": 3, "nbr": 4}[plane]
    c = 0 if where == 0 else len(bad) - 1
    arr = np.array(bad[c][idx], np.int64, copy=True)
    arr.reshape(-1)[where] = -1 if plane == "snk" else CAP_MAX + 1
    bad[c][idx] = arr
    if i32:
        arr = arr.astype(np.int32)
        bad[c][idx] = arr
    with pytest.raises(CapacityOverflowError):
        engine.solve_composites([tuple(b) for b in bad], i32=i32)
    got = engine.solve_composites([tuple(it) for it in items], i32=i32)
    for (w, h, src, snk, nbr, _), (flow, lab) in zip(items, got):
        f, want, _ = oracle.solve(w, h, np.asarray(src, np.int64), np.asarray(snk, np.int64),
                                  np.asarray(nbr, np.int64).reshape(-1), [])
        assert flow == f and np.array_equal(lab, want)


def test_large_grid_properties(engine):
    """C4-shaped single lambda (1920x1080): certificate checks that do not
    need the reference -- the labels' cut cost equals the flow, and the
    masks are nested along the schedule."""
    p = synth.generate(1920, 1080, rng_seed=0).problems[0]
    sched = LambdaSchedule((1, 7, 24))
    res = solve_seed_supergraph([p], sched)
    want = {1: 20920322, 7: 44135775, 24: 44904079}   # SURVEY.md Appendix A (scipy oracle)
    prev = None
    from paper_1509_06004_b200 import instantiate
    for lam, c in zip(sched, res.cuts):
        assert c.flow == want[lam]
        assert cut_cost(instantiate(p, lam), c.labels) == c.flow
        if prev is not None:
            assert not (prev & ~c.labels.astype(bool)).any()
        prev = c.labels.astype(bool)


@pytest.mark.parametrize("persistent", [0, 1])
def test_c1_stress_repeated(engine, persistent):
    """Worklist/queue races show up as rare label or flow differences:
    repeat the C1 supergraph in both scheduling modes."""
    from paper_1509_06004_b200 import _native
    g = load_synth("c1_160x120.npz")
    probs = synth.generate(160, 120, rng_seed=0).problems
    s = _native.Solver(0, persistent=persistent)
    try:
        for rep in range(12):
            _, flows, labels = s.solve_seed_batch(160, 120, probs, g["lambdas"], "auto")
            assert flows[0].tolist() == g["flows"], rep
            for j in range(20):
                assert np.array_equal(labels[0][j], g["labels"][j]), (rep, j)
    finally:
        s.close()


@pytest.mark.parametrize("mode", ["async", "rolling", "steps"])
@pytest.mark.parametrize("chain", [2, 3, 5])
def test_warm_start_chains_match_reference(engine, chain, mode):
    """Warm start along the nested schedule (each grid solves `chain`
    consecutive lambdas, reusing the previous maximum preflow) must give the
    reference's cuts, swapped families included -- both with a common step
    per lambda (rolling=0) and with every grid advancing as soon as it
    finishes (rolling=1)."""
    from paper_1509_06004_b200 import _native
    s = _native.Solver(0, chain=chain, **{"async": int(mode == "async")}, rolling=int(mode == "rolling"))
    try:
        for case in load_seed_supergraphs():
            probs = _problems(case)
            sw, flows, labels = s.solve_seed_batch(case["width"], case["height"], probs,
                                                   case["lambdas"], case["mode"])
            assert [bool(x) for x in sw for _ in case["lambdas"]] == case["swapped"]
            assert flows.reshape(-1).tolist() == case["flows"]
            assert [l.tolist() for l in labels.reshape(len(case["flows"]), -1)] == case["labels"]
        g = load_synth("c1_160x120.npz")
        probs = synth.generate(160, 120, rng_seed=0).problems
        for mode in ("auto", "on"):
            _, flows, labels = s.solve_seed_batch(160, 120, probs, g["lambdas"], mode)
            assert flows[0].tolist() == g["flows"]
            for j in range(20):
                assert np.array_equal(labels[0][j], g["labels"][j]), (mode, j)
        # steps: common lambda steps (rolling=0) / label rounds (rolling=1) /
        # lambda-graphs finished (asynchronous solver)
        st = s.stats()
        if mode == "async":
            assert st["async_mode"] and st["steps"] == 20
        else:
            assert st["steps"] == chain if mode == "steps" else st["steps"] >= chain
    finally:
        s.close()


def test_c3_cpmc_image_rolling_vs_cold_vs_reference(engine):
    """C3 CPMC image (500x375, 25 seeds x types A/B x L20): the rolling warm
    start (default for many problems) must reproduce the cold per-lambda
    solve bit for bit, the reference's per-type flow sums (SURVEY.md
    Appendix A: A 2,408,913,070, B 2,293,473,574; first seed A 101,007,728,
    B 99,225,144) and the oracle's cuts on sampled (problem, lambda) pairs."""
    from paper_1509_06004_b200 import _native
    b = synth.generate(500, 375, 5, 5, rng_seed=0, types=("A", "B"))
    lams = synth.L20
    warm = _native.Solver(0)
    cold = _native.Solver(0, chain=1)
    try:
        _, fw, lw = warm.solve_seed_batch(500, 375, b.problems, lams, "auto")
        assert warm.stats()["cycles"] > 0
        _, fc, lc = cold.solve_seed_batch(500, 375, b.problems, lams, "auto")
    finally:
        warm.close()
        cold.close()
    assert np.array_equal(fw, fc)
    assert np.array_equal(lw, lc)
    per = fw.sum(axis=1)
    assert int(per[0::2].sum()) == 2408913070 and int(per[1::2].sum()) == 2293473574
    assert int(per[0]) == 101007728 and int(per[1]) == 99225144
    rng = np.random.default_rng(303)
    picks = [(0, 0), (17, 9), (49, 19)] + [(int(rng.integers(0, 50)), int(rng.integers(0, 20)))
                                           for _ in range(37)]
    jobs = []
    for pi, li in picks:
        p = b.problems[pi]
        src, snk, nbr = oracle.instantiate(p.unary_base, p.unary_slope, p.sink_base, p.pairwise,
                                           p.fg_seeds, p.bg_seeds, lams[li])
        jobs.append((500, 375, src, snk, nbr, None))
    for (pi, li), (flow, labels, _) in zip(picks, oracle.solve_many(jobs)):
        assert int(fw[pi, li]) == flow, (pi, li)
        assert np.array_equal(lw[pi, li].reshape(-1), labels), (pi, li)


def test_c5_batch_sampled_cuts_vs_oracle(engine):
    """C5's unit of work -- 32 distinct CPMC images (rng_seed 0..31) in one
    device batch, 1,600 warm-start chains, the step-synchronous rolling
    engine the bench runs -- against the oracle on 50 sampled (image,
    problem, lambda) cuts: bit-exact flows and masks.  Every cut also passed
    the device certificate (cut cost == flow) inside the solve."""
    from paper_1509_06004_b200 import _native
    probs = []
    for i in range(32):
        probs += synth.generate(500, 375, 5, 5, rng_seed=i, types=("A", "B")).problems
    s = _native.Solver(0)
    try:
        _, fl, lab = s.solve_seed_batch(500, 375, probs, synth.L20, "auto")
        assert s.stats()["async_mode"] == 0   # 32 images: the step-synchronous engine
    finally:
        s.close()
    rng = np.random.default_rng(2026)
    picks = [(int(rng.integers(0, len(probs))), int(rng.integers(0, len(synth.L20)))) for _ in range(50)]
    jobs = []
    for pi, li in picks:
        p = probs[pi]
        src, snk, nbr = oracle.instantiate(p.unary_base, p.unary_slope, p.sink_base, p.pairwise,
                                           p.fg_seeds, p.bg_seeds, synth.L20[li])
        jobs.append((500, 375, src, snk, nbr, None))
    for (pi, li), (flow, labels, _) in zip(picks, oracle.solve_many(jobs)):
        assert int(fl[pi, li]) == flow, (pi // 50, pi % 50, li)
        assert np.array_equal(lab[pi, li].reshape(-1), labels), (pi // 50, pi % 50, li)


def test_staging_shares_equal_planes_but_checks_each_mask(engine):
    """Problems with equal unary/sink planes are staged once (pointer-equal
    or content-equal arrays); results stay per problem, and each problem's
    range check still uses its own seed masks."""
    from paper_1509_06004_b200 import _native
    from paper_1509_06004_b200.grid import CapacityOverflowError
    b = synth.generate(64, 48, 1, 2, rng_seed=3, types=("A", "B"))
    a0, b0 = b.problems[0], b.problems[1]
    assert a0.unary_base.ctypes.data == b0.unary_base.ctypes.data   # generator shares the seed terms
    # a content-equal copy with the other seed type must give the same cuts as b0
    c0 = SeedProblem(64, 48, a0.unary_base.copy(), a0.unary_slope.copy(), a0.sink_base.copy(),
                     a0.pairwise, a0.fg_seeds, b0.bg_seeds)
    lams = [1, 4, 9]
    s = _native.Solver(0)
    try:
        _, f1, l1 = s.solve_seed_batch(64, 48, [a0, b0, b.problems[2]], lams, "auto")
        _, f2, l2 = s.solve_seed_batch(64, 48, [a0, c0, b.problems[2]], lams, "auto")
        assert np.array_equal(f1, f2) and np.array_equal(l1, l2)
        for pi, p in enumerate((a0, b0)):
            for li, lam in enumerate(lams):
                src, snk, nbr = oracle.instantiate(p.unary_base, p.unary_slope, p.sink_base, p.pairwise,
                                                   p.fg_seeds, p.bg_seeds, lam)
                flow, labels, _ = oracle.solve(64, 48, src, snk, nbr)
                assert int(f1[pi, li]) == flow and np.array_equal(l1[pi, li], labels)
        # pixel 0 is a bg seed of type A only: an out-of-range sink term there
        # is exempt for A but must be rejected for the plane-sharing B problem
        sink = a0.sink_base.copy()
        sink[0] = CAP_MAX + 1
        pa = SeedProblem(64, 48, a0.unary_base, a0.unary_slope, sink, a0.pairwise, a0.fg_seeds,
                         a0.bg_seeds)
        pb = SeedProblem(64, 48, a0.unary_base, a0.unary_slope, sink, a0.pairwise, a0.fg_seeds,
                         b0.bg_seeds - {0})
        s.solve_seed_batch(64, 48, [pa], lams, "off")
        with pytest.raises(CapacityOverflowError):
            s.solve_seed_batch(64, 48, [pa, pb], lams, "off")
    finally:
        s.close()


def test_async_solver_matches_step_synchronous_under_load(engine):
    """The asynchronous solver (every grid on its own phase machine in one
    persistent kernel) against the step-synchronous engine on a loaded batch
    (4 CPMC images, 200 warm-start chains), repeated: bit-identical flows and
    masks, integrity check on.  Guards the hand-off / phase-transition races
    (a drained-discharge early finish once passed small tests and failed
    here)."""
    from paper_1509_06004_b200 import _native
    probs = []
    for i in range(4):
        probs += synth.generate(500, 375, 5, 5, rng_seed=i, types=("A", "B")).problems
    sync = _native.Solver(0, **{"async": 0})
    asy = _native.Solver(0, **{"async": 1})
    flush = _native.Solver(0, **{"async": 1}, push_flush=8)   # mid-pass hand-off variant
    try:
        _, fs, ls = sync.solve_seed_batch(500, 375, probs, synth.L20, "auto")
        for s in (asy, asy, flush):
            _, fa, la = s.solve_seed_batch(500, 375, probs, synth.L20, "auto")
            assert s.stats()["async_mode"] == 1
            assert np.array_equal(fa, fs)
            assert np.array_equal(la, ls)
    finally:
        sync.close()
        asy.close()
        flush.close()


def test_device_scoring_matches_reference():
    """Device scoring (pmf_seed_score) of a seed supergraph equals the
    reference's per-cut foreground counts and exact overlaps
    (harness/bench.py:104-111), and the host overlap of the returned masks."""
    from fractions import Fraction
    from conftest import load_scores
    from paper_1509_06004_b200.scoring import overlap
    g = load_scores()
    b = synth.generate(g["width"], g["height"], g["rows"], g["cols"], rng_seed=g["rng_seed"])
    res = solve_seed_supergraph(b.problems, LambdaSchedule(g["lambdas"]), "auto", truths=b.truths)
    K = len(g["lambdas"])
    assert len(res.scores) == len(b.problems) * K
    for pi, rec in enumerate(g["problems"]):
        for j in range(K):
            cut, sc = res.cuts[pi * K + j], res.scores[pi * K + j]
            assert cut.flow == rec["flows"][j]
            assert sc.foreground == rec["foreground"][j] == int(cut.labels.sum())
            assert sc.overlap == Fraction(*rec["overlap"][j]) == overlap(cut.labels, b.truths[pi])


def test_seed_supergraph_stream_matches_single_calls():
    """solve_seed_supergraphs (stager / runner / fetch overlap over two
    solvers) returns exactly what solve_seed_supergraph returns per batch --
    flows, label masks, layouts, device scores -- including a mixed-width
    batch (solved inline) and a failing batch (raised at its position)."""
    from paper_1509_06004_b200 import solve_seed_supergraphs
    from paper_1509_06004_b200.supergraph import SupergraphError
    sched = LambdaSchedule(synth.L20[:6])
    imgs = [synth.generate(160, 120, 2, 2, rng_seed=s, types=("A", "B")) for s in range(4)]
    batches = [b.problems for b in imgs[:3]]
    mixed = synth.generate(96, 120, 1, 1, rng_seed=9).problems + imgs[3].problems[:2]
    batches.append(mixed)
    truths = [b.truths for b in imgs[:3]] + [None]
    want = [solve_seed_supergraph(b, sched, "auto", truths=t) for b, t in zip(batches, truths)]
    got = list(solve_seed_supergraphs(batches, sched, "auto", truths=truths))
    assert len(got) == len(want)
    for g, w in zip(got, want):
        assert g.layout == w.layout
        assert [c.flow for c in g.cuts] == [c.flow for c in w.cuts]
        assert all(np.array_equal(a.labels, b.labels) for a, b in zip(g.cuts, w.cuts))
        assert g.scores == w.scores
    out = []
    with pytest.raises(SupergraphError):
        for r in solve_seed_supergraphs([batches[0], [], batches[1]], sched):
            out.append(r)
    assert len(out) == 1 and [c.flow for c in out[0].cuts] == [c.flow for c in want[0].cuts]


def test_run_dynamic_on_gpu_backend():
    """scheduler.py:253-292 policy over the GPU backend (one executor per
    device, queued tasks coalesced into device batches): composite tasks and
    device-built seed-supergraph tasks in one run give the same cuts as the
    direct calls, which are pinned to the reference elsewhere."""
    from paper_1509_06004_b200 import GpuBackend, Task, gpu_workers, run_dynamic
    b = synth.generate(160, 120, 2, 2, rng_seed=1)
    sched = LambdaSchedule(synth.L20[:6])
    tasks = []
    for i, p in enumerate(b.problems):
        comp, layout, _ = build_seed_supergraph([p], sched, "auto")
        tasks.append(Task(id=2 * i, graph=comp, layout=layout, duration=comp.n))
        tasks.append(Task(id=2 * i + 1, problems=(p,), schedule=sched))
    backend = GpuBackend(max_batch=3)
    try:
        schedule, cuts = run_dynamic(tasks, gpu_workers([0], slots=3), backend)
    finally:
        backend.close()
    assert sorted(r.task_id for r in schedule.records) == [t.id for t in tasks]
    for i, p in enumerate(b.problems):
        comp, layout, originals = build_seed_supergraph([p], sched, "auto")
        direct = solve_composite(comp, layout)
        assert cuts[2 * i].flow == direct.flow and np.array_equal(cuts[2 * i].labels, direct.labels)
        parts = split(layout, direct, originals)
        dev = cuts[2 * i + 1]
        assert [c.flow for c in dev.cuts] == [c.flow for c in parts]
        assert all(np.array_equal(a.labels, c.labels) for a, c in zip(dev.cuts, parts))


def test_run_dynamic_streams_coalesced_seed_tasks():
    """Seed-supergraph tasks coalesced on one GPU run as a batch stream
    (GpuBackend._run_batch -> solve_seed_supergraphs); every task's result
    equals the direct call, a task with another schedule forms its own group."""
    from paper_1509_06004_b200 import GpuBackend, Task, gpu_workers, run_dynamic
    sched, other = LambdaSchedule(synth.L20[:5]), LambdaSchedule(synth.L20[2:6])
    probs = [synth.generate(120, 90, 1, 2, rng_seed=s, types=("A", "B")).problems for s in range(6)]
    tasks = [Task(id=i, problems=tuple(p), schedule=sched if i != 4 else other) for i, p in enumerate(probs)]
    backend = GpuBackend(max_batch=6)
    try:
        schedule, cuts = run_dynamic(tasks, gpu_workers([0], slots=6), backend)
    finally:
        backend.close()
    assert sorted(r.task_id for r in schedule.records) == list(range(6))
    for t in tasks:
        want = solve_seed_supergraph(list(t.problems), t.schedule)
        got = cuts[t.id]
        assert got.layout == want.layout
        assert [c.flow for c in got.cuts] == [c.flow for c in want.cuts]
        assert all(np.array_equal(a.labels, b.labels) for a, b in zip(got.cuts, want.cuts))


@pytest.mark.parametrize("mode", [1, 0])
def test_seed_batches_on_edge_shapes(engine, mode):
    """Seed batches through the device builder on odd shapes (1xN, Nx1,
    tiles straddling 32-px boundaries), warm chains and cold grids, both
    schedulers (mode 1: asynchronous kernel, 0: step-synchronous), against
    the oracle's restatement of the reference solver per (problem, lambda)."""
    from paper_1509_06004_b200 import _native
    rng = np.random.default_rng(11)
    lams = [1, 3, 8, 20]
    # W % 4 == 0 shapes take the 4-pixel-group certificate kernel
    for (w, h) in [(1, 7), (9, 1), (33, 2), (31, 33), (65, 34), (4, 5), (8, 1), (36, 3), (64, 33)]:
        n = w * h
        probs = []
        for k in range(9):   # >= warm_min_problems: warm-start chains
            nb = rng.integers(1, 20, (4, h, w))
            nb[0][:, 0] = 0
            nb[1][:, -1] = 0
            nb[2][0, :] = 0
            nb[3][-1, :] = 0
            fg = {int(rng.integers(0, n))}
            bg = {int(x) for x in rng.integers(0, n, 2)} - fg
            probs.append(SeedProblem(w, h, rng.integers(0, 10, n), rng.integers(0, 4, n),
                                     rng.integers(0, 25, n), nb.reshape(4, n), fg, bg))
        for chain in (0, 1):
            s = _native.Solver(0, chain=chain, **{"async": mode})
            try:
                sw, flows, labels = s.solve_seed_batch(w, h, probs, lams, "auto")
            finally:
                s.close()
            for pi, p in enumerate(probs):
                for li, lam in enumerate(lams):
                    src, snk, nbr = oracle.instantiate(p.unary_base, p.unary_slope, p.sink_base, p.pairwise,
                                                       p.fg_seeds, p.bg_seeds, lam)
                    # swapped families decode to the original graph's cut
                    # (swap invariance, test_acceptance.py:79-87)
                    f, lab, _ = oracle.solve(w, h, src, snk, nbr)
                    assert int(flows[pi, li]) == f, (w, h, chain, pi, lam)
                    assert np.array_equal(labels[pi, li], lab), (w, h, chain, pi, lam)


@pytest.mark.parametrize("mode", [1, 0])
def test_c4_all_lambdas_both_schedulers(engine, mode):
    """C4 (1920x1080, lambdas 1..24): every per-lambda flow of SURVEY.md
    Appendix A (scipy-Dinic oracle, reference-confirmed at 1, 7, 24) and the
    foreground counts, through the asynchronous kernel (mode 1) and the
    step-synchronous engine (mode 0)."""
    from paper_1509_06004_b200 import _native
    p = synth.generate(1920, 1080, rng_seed=0).problems
    lams = synth.C4_LAMBDAS
    flows_a = [20920322, 25439507, 29721283, 37249143, 44135775, 44603555, 44719143, 44904079]
    fg_a = [611418, 986561, 1015195, 1180813, 1180813, 2067603, 2067604, 2067604]
    s = _native.Solver(0, **{"async": mode})
    try:
        _, flows, labels = s.solve_seed_batch(1920, 1080, p, lams, "auto")
        assert s.stats()["async_mode"] == mode
    finally:
        s.close()
    assert flows[0].tolist() == flows_a
    assert [int(l.sum()) for l in labels[0]] == fg_a


@pytest.mark.parametrize("mode,vec", [(0, 1), (1, 1), (1, 0)])
def test_integrity_check_catches_a_corrupted_cut(engine, mode, vec):
    """The device certificate (cut cost of every emitted mask == its flow,
    grid.py:159-178 / supergraph.py:181-186) rejects a batch whose emitted
    mask was corrupted (knob verify=2 flips one label before the check), in
    both schedulers and with both certificate kernels (verify_vec: 4-pixel
    groups, W % 4 == 0 here, or per pixel); the same batch passes with
    verify=1."""
    from paper_1509_06004_b200 import _native
    from paper_1509_06004_b200.solvers import NonMaximalFlowError
    probs = synth.generate(500, 375, 2, 2, rng_seed=3, types=("A", "B")).problems
    for verify in (1, 2):
        s = _native.Solver(0, **{"async": mode}, verify=verify, verify_vec=vec)
        try:
            if verify == 1:
                s.solve_seed_batch(500, 375, probs, synth.L20, "auto")
            else:
                with pytest.raises(NonMaximalFlowError, match="integrity"):
                    s.solve_seed_batch(500, 375, probs, synth.L20, "auto")
        finally:
            s.close()


@pytest.mark.parametrize("split", [1, 0])
def test_composite_span_split_vs_oracle(engine, split):
    """Composites as one grid per isolated segment span (knob comp_split=1)
    or one grid per composite: flows and labels equal the oracle's
    (supergraph.py:190-207 semantics), for join()-built composites (zero
    bridges: split) and for leaky ones -- a bridge pixel with a terminal
    capacity, an arc across a span boundary -- which must not be split."""
    from paper_1509_06004_b200 import _native
    rng = np.random.default_rng(91)
    items, ref = [], []
    for case in range(10):
        h = int(rng.integers(3, 40))
        graphs = []
        for _ in range(int(rng.integers(2, 5))):
            w = int(rng.integers(1, 40))
            nb = rng.integers(0, 30, (4, h, w))
            nb[0][:, 0] = 0
            nb[1][:, -1] = 0
            nb[2][0, :] = 0
            nb[3][-1, :] = 0
            graphs.append(grid(w, h, rng.integers(0, 60, w * h), rng.integers(0, 60, w * h), nb.reshape(4, -1)))
        flags = [bool(rng.integers(0, 2)) for _ in graphs]
        comp, lay = join([apply_swap(g) if f else g for g, f in zip(graphs, flags)], swapped=flags)
        src, snk = comp.src_cap.copy(), comp.snk_cap.copy()
        nbr = comp.nbr_cap.copy().reshape(4, comp.height, comp.width)
        seg0 = lay.segments[0]
        if case % 3 == 1 and lay.bridge_columns:     # a bridge pixel with a source arc
            src.reshape(comp.height, comp.width)[h // 2, lay.bridge_columns[0]] = 7
        if case % 3 == 2:                            # an arc leaving the first span
            nbr[1][h // 2, seg0.offset + seg0.width - 1] = 9
        segs = [(s.offset, s.width, s.swapped) for s in lay.segments]
        items.append((comp.width, comp.height, src, snk, nbr.reshape(4, -1), segs))
        ref.append(oracle.solve(comp.width, comp.height, src, snk, nbr.reshape(4, -1), segs))
    s = _native.Solver(0, comp_split=split)
    try:
        got = s.solve_composites(items)
    finally:
        s.close()
    for (f, lab), (rf, rlab, _) in zip(got, ref):
        assert f == rf
        assert np.array_equal(lab, rlab)


def test_composite_bits_from_device(engine):
    """pmf_composite_bits: the labels of each composite of the last solve,
    packed on the device in the wire's LSB-first order, equal the packed
    byte labels; composites solved with labels left on the device still
    report their flows."""
    from paper_1509_06004_b200 import _native
    from paper_1509_06004_b200.wire import pack_bits
    rng = np.random.default_rng(5)
    items = []
    for (w, h) in [(7, 5), (33, 17), (64, 40), (3, 1)]:
        nb = rng.integers(0, 20, (4, h, w))
        nb[0][:, 0] = 0
        nb[1][:, -1] = 0
        nb[2][0, :] = 0
        nb[3][-1, :] = 0
        items.append((w, h, rng.integers(0, 40, w * h), rng.integers(0, 40, w * h), nb.reshape(4, -1), None))
    s = _native.Solver(0)
    try:
        ref = s.solve_composites(items)
        got = s.solve_composites(items, labels=False)
        assert [f for f, _ in got] == [f for f, _ in ref] and all(l is None for _, l in got)
        for c, (w, h, *_ ) in enumerate(items):
            assert s.composite_bits(c, w * h) == pack_bits(ref[c][1])
    finally:
        s.close()


# every tuning knob that survives on the ABI (pmf_solver_set), each value
# against the reference's C1 cuts (golden) -- the knob must not change results
KNOB_CASES = [
    {"graph": 0}, {"graph": 0, "async": 0}, {"async": 0}, {"async": 1},
    {"async": 0, "persistent": 0}, {"async": 0, "persistent_bfs": 1}, {"async": 0, "bfs_multi": 0},
    {"async": 0, "rolling": 0}, {"chain": 1}, {"chain": 5}, {"chain": 5, "async": 0},
    {"fresh_skip": 0}, {"warp": 0}, {"warp": 0, "async": 0}, {"async_cont": 0}, {"async_prefetch": 0},
    {"async_spec": 0}, {"adv_keep_h": 0}, {"push_iters": 4}, {"relabel_every": 0},
    {"relabel_every": 3, "async": 0}, {"push_budget": 1, "async": 0}, {"push_budget_warm": 1, "chain": 20},
    {"push_budget_add": 0}, {"push_sweeps": 2, "async": 0, "persistent": 0}, {"bfs_chunk": 1, "graph": 0},
    {"push_flush": 8}, {"verify_vec": 0}, {"timing": 1}, {"wide_pulses": 8, "force_wide": 1},
    {"warm_min_problems": 1}, {"async_max_tiles": 0}, {"async_max_grid_tiles": 0},
    {"phase_log": 1}, {"max_cycles": 100000},
]


@pytest.mark.parametrize("knobs", KNOB_CASES, ids=lambda k: ",".join(f"{a}={b}" for a, b in k.items()))
def test_every_knob_keeps_c1_bit_exact(engine, knobs):
    from paper_1509_06004_b200 import _native
    gold = load_synth("c1_160x120.npz")
    batch = synth.generate(160, 120, 1, 1, rng_seed=0)
    s = _native.Solver(0, **knobs)
    try:
        _, fl, lab = s.solve_seed_batch(160, 120, batch.problems, gold["lambdas"], "auto")
    finally:
        s.close()
    assert [int(f) for f in fl[0]] == gold["flows"]
    for k in range(len(gold["flows"])):
        assert np.array_equal(lab[0, k], gold["labels"][k])


def test_removed_knobs_are_refused(engine):
    """Measured-and-rejected variants are gone from the ABI."""
    from paper_1509_06004_b200 import _native
    s = _native.Solver(0)
    try:
        for name, v in (("push_mode", 1), ("relax_cap", 4), ("push_minb", 1), ("grid_div", 2), ("warp", 1),
                        ("warp", 2), ("warp_bfs_tiles", 5)):
            with pytest.raises(ValueError):
                s.set(name, v)
    finally:
        s.close()
