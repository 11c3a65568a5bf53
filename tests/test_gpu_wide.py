"""The int64 state variant (csrc/wide.cuh): every graph the reference admits
(grid.py:102-130: capacities in [0, CAP_MAX], total < 2^62) solves, bit-exact
against the oracle, including graphs whose excess leaves int32 (CAP_MAX arc
pairs, CAP_MAX seeds beside CAP_MAX arcs).  The wire frames of this kind
(tests/golden/wire_frames.json, wide_*) are answered OK by serve_payload in
test_wire.py."""

import numpy as np
import pytest

import oracle
from paper_1509_06004_b200 import (CAP_MAX, GridGraph, LambdaSchedule, SeedProblem, _native, admit,
                                   apply_swap, cut_cost, join, maxflow_many, solve_composites,
                                   solve_seed_supergraph, synth)

pytestmark = pytest.mark.gpu


def zero_border(nb):
    nb[0][:, 0] = 0
    nb[1][:, -1] = 0
    nb[2][0, :] = 0
    nb[3][-1, :] = 0
    return nb


def wide_caps(rng, shape):
    """{0, small, up to CAP_MAX, CAP_MAX} mixture (make_wire_golden.wide_grid)."""
    kind = rng.integers(0, 4, shape)
    return np.where(kind == 0, 0, np.where(kind == 1, rng.integers(1, 100, shape),
                                           np.where(kind == 2, rng.integers(1, CAP_MAX + 1, shape),
                                                    CAP_MAX))).astype(np.int64)


def wide_graph(rng, w, h, draw=wide_caps):
    nb = zero_border(draw(rng, (4, h, w)))
    return admit(GridGraph(w, h, draw(rng, w * h), draw(rng, w * h), nb.reshape(4, -1)))


def uniform_caps(rng, shape):
    return rng.integers(0, CAP_MAX + 1, shape).astype(np.int64)


def check(graphs, got):
    for g, r in zip(graphs, got):
        f, lab, _ = oracle.solve(g.width, g.height, g.src_cap, g.snk_cap, g.nbr_cap)
        assert r.flow == f
        assert np.array_equal(r.labels, lab)
        assert cut_cost(g, r.labels) == r.flow


def test_capmax_mixture_graphs_vs_oracle(engine):
    rng = np.random.default_rng(31)
    graphs = [wide_graph(rng, int(rng.integers(1, 40)), int(rng.integers(1, 40))) for _ in range(30)]
    got = maxflow_many(graphs)
    assert _native.solver_for_thread(0).stats()["wide_mode"] == 1
    check(graphs, got)


def test_uniform_caps_up_to_2_30_vs_oracle(engine):
    rng = np.random.default_rng(32)
    graphs = [wide_graph(rng, int(rng.integers(2, 64)), int(rng.integers(2, 48)), uniform_caps)
              for _ in range(12)]
    check(graphs, maxflow_many(graphs))


def test_capmax_interior_arc_pairs_and_seeds(engine):
    """Every interior arc at CAP_MAX, CAP_MAX terminals on a few pixels."""
    rng = np.random.default_rng(33)
    graphs = []
    for (w, h) in ((33, 17), (64, 64), (5, 70)):
        nb = zero_border(np.full((4, h, w), CAP_MAX, np.int64))
        src = np.zeros(w * h, np.int64)
        snk = np.zeros(w * h, np.int64)
        src[rng.choice(w * h, 3, replace=False)] = CAP_MAX
        snk[rng.choice(w * h, 3, replace=False)] = CAP_MAX
        snk = np.where(snk == 0, rng.integers(0, 3, w * h), snk)
        graphs.append(admit(GridGraph(w, h, src, snk, nb.reshape(4, -1))))
    check(graphs, maxflow_many(graphs))


def test_wide_composites_with_swapped_spans(engine):
    rng = np.random.default_rng(34)
    tasks, ref = [], []
    for _ in range(6):
        h = int(rng.integers(3, 30))
        parts = [wide_graph(rng, int(rng.integers(2, 30)), h) for _ in range(int(rng.integers(1, 4)))]
        sw = [bool(rng.integers(0, 2)) for _ in parts]
        comp, lay = join([apply_swap(g) if s else g for g, s in zip(parts, sw)], swapped=sw)
        tasks.append((comp, lay))
        ref.append(oracle.solve(comp.width, comp.height, comp.src_cap, comp.snk_cap, comp.nbr_cap,
                                [(s.offset, s.width, s.swapped) for s in lay.segments]))
    for r, (f, lab, _) in zip(solve_composites(tasks), ref):
        assert r.flow == f and np.array_equal(r.labels, lab)


def test_force_wide_reproduces_c1(engine):
    """The int64 variant on an ordinary batch (knob force_wide): C1's
    per-lambda cuts equal the reference's (tests/golden/c1_160x120.npz)."""
    from conftest import load_synth
    gold = load_synth("c1_160x120.npz")
    batch = synth.generate(160, 120, 1, 1, rng_seed=0)
    s = _native.solver_for_thread(0)
    s.set("force_wide", 1)
    try:
        res = solve_seed_supergraph(batch.problems, LambdaSchedule(gold["lambdas"]), "auto")
        assert s.stats()["wide_mode"] == 1
    finally:
        s.set("force_wide", 0)
    assert [c.flow for c in res.cuts] == gold["flows"]
    for k, c in enumerate(res.cuts):
        assert np.array_equal(c.labels, gold["labels"][k])
    assert res.flow == 27814225


def capmax_block(p, x0, y0, k):
    """p with every arc inside the k x k block at (x0, y0) at CAP_MAX (arcs
    at CAP_MAX are outside instantiate's finite-capacity budget,
    parametric.py:160-165, so the family stays admissible)."""
    W, H = p.width, p.height
    pw = p.pairwise.reshape(4, H, W).copy()
    pw[0, y0:y0 + k, x0 + 1:x0 + k] = CAP_MAX   # LEFT arcs staying in the block
    pw[1, y0:y0 + k, x0:x0 + k - 1] = CAP_MAX   # RIGHT
    pw[2, y0 + 1:y0 + k, x0:x0 + k] = CAP_MAX   # UP
    pw[3, y0:y0 + k - 1, x0:x0 + k] = CAP_MAX   # DOWN
    return SeedProblem(W, H, p.unary_base, p.unary_slope, p.sink_base, pw.reshape(4, -1),
                       p.fg_seeds, p.bg_seeds)


def test_wide_seed_batch_vs_oracle(engine):
    """CAP_MAX seeds beside CAP_MAX arcs: a seed family with a block of
    CAP_MAX arcs around its foreground seed takes the int64 variant
    (8 x max arc pair > 2^31) instead of raising CapacityOverflowError; every
    (problem, lambda) cut equals the oracle's, swapped families included."""
    b = synth.generate(48, 36, 2, 1, rng_seed=3, types=("A", "B"))
    probs = []
    for (x, y), p in zip([c for c in b.coords for _ in b.types], b.problems):
        probs.append(capmax_block(p, x - 3, y - 3, 7))
    sched = LambdaSchedule((1, 5, 40, 300))
    for mode in ("auto", "on"):
        res = solve_seed_supergraph(probs, sched, mode)
        assert _native.solver_for_thread(0).stats()["wide_mode"] == 1
        k = 0
        for p in probs:
            for lam in sched:
                src, snk, nbr = oracle.instantiate(p.unary_base, p.unary_slope, p.sink_base, p.pairwise,
                                                   p.fg_seeds, p.bg_seeds, lam)
                f, lab, _ = oracle.solve(p.width, p.height, src, snk, nbr)
                assert res.cuts[k].flow == f
                assert np.array_equal(res.cuts[k].labels, lab)
                k += 1


def test_wide_integrity_hook(engine):
    """verify=2 corrupts one emitted label of a wide seed batch: the device
    certificate must catch it (NonMaximalFlowError)."""
    from paper_1509_06004_b200 import NonMaximalFlowError
    b = synth.generate(48, 36, 1, 1, rng_seed=4)
    s = _native.solver_for_thread(0)
    s.set("force_wide", 1)
    s.set("verify", 2)
    try:
        with pytest.raises(NonMaximalFlowError):
            solve_seed_supergraph(b.problems, LambdaSchedule((1, 9)), "off")
    finally:
        s.set("verify", 1)
        s.set("force_wide", 0)


def test_composite_solve_invalidates_the_staged_seed_batch(engine):
    """A composite solve overwrites the staged batch's device buffers: the
    seed run / fetch must refuse instead of returning wrong results."""
    b = synth.generate(40, 30, 1, 1, rng_seed=5)
    s = _native.Solver(0)
    try:
        s.seed_stage(40, 30, b.problems, (1, 2, 3))
        s.seed_run()
        g = wide_graph(np.random.default_rng(1), 9, 7)
        s.solve_composites([(g.width, g.height, g.src_cap, g.snk_cap, g.nbr_cap, None)])
        with pytest.raises(ValueError):
            s.seed_run()
        with pytest.raises(ValueError):
            s.seed_fetch()
    finally:
        s.close()


@pytest.mark.parametrize("wide", [0, 1])
def test_composite_certificate_catches_a_corrupted_cut(engine, wide):
    """Composite solves carry the device certificate too (cut cost of the
    emitted labels == flow, supergraph.py:181-186, rpc.py:328-331): with the
    verify=2 hook corrupting one label the solve raises; without it the same
    composites pass."""
    from paper_1509_06004_b200 import NonMaximalFlowError
    rng = np.random.default_rng(40 + wide)
    parts = [wide_graph(rng, 12, 9) if wide else
             admit(GridGraph(12, 9, rng.integers(0, 50, 108), rng.integers(0, 50, 108),
                             zero_border(rng.integers(1, 30, (4, 9, 12))).reshape(4, -1)))
             for _ in range(3)]
    comp, lay = join([parts[0], apply_swap(parts[1]), parts[2]], swapped=[False, True, False])
    s = _native.solver_for_thread(0)
    good = solve_composites([(comp, lay)])[0]
    assert s.stats()["wide_mode"] == wide
    assert cut_cost(comp, good.labels) == good.flow
    s.set("verify", 2)
    try:
        with pytest.raises(NonMaximalFlowError):
            solve_composites([(comp, lay)])
    finally:
        s.set("verify", 1)
