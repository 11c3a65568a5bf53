"""Host-side API (no GPU): admission, knitting, swap algebra, schedules,
seed-problem checks and the dynamic scheduler policy, each against the
reference's golden vectors or its documented semantics."""

import numpy as np
import pytest

import oracle
from conftest import load_composites, load_seed_supergraphs
from paper_1509_06004_b200 import (CAP_MAX, BatchAborted, BorderEdgeError, CapacityOverflowError,
                                   CutResult, GridGraph, LambdaSchedule, NegativeCapacityError,
                                   ProblemError, ScheduleError, SeedProblem, ShapeError,
                                   SupergraphError, Task, ThreadedBackend, WorkerHandle, admit,
                                   apply_swap, build_seed_supergraph, cut_cost, instantiate, join,
                                   run_dynamic, split, swap_decision, terminal_balance)
from paper_1509_06004_b200.parametric import check_family
from paper_1509_06004_b200.supergraph import check_seed_supergraph, seed_layout


def mk(w, h, src=0, snk=0, left=0, right=0, up=0, down=0):
    n = w * h

    def full(v):
        return np.full(n, v, np.int64) if np.isscalar(v) else np.asarray(v, np.int64).reshape(-1).copy()

    nb = np.stack([full(left), full(right), full(up), full(down)]).reshape(4, h, w)
    nb[0][:, 0] = nb[1][:, -1] = 0
    nb[2][0, :] = nb[3][-1, :] = 0
    return admit(GridGraph(w, h, full(src), full(snk), nb.reshape(4, n)))


# ------------------------------------------------------------------ grid

def test_admit_error_classes():
    with pytest.raises(NegativeCapacityError):
        admit(GridGraph(2, 1, [-1, 0], [0, 0], np.zeros((4, 2))))
    with pytest.raises(CapacityOverflowError):
        admit(GridGraph(2, 1, [CAP_MAX + 1, 0], [0, 0], np.zeros((4, 2))))
    nb = np.zeros((4, 2), np.int64)
    nb[0, 0] = 1  # LEFT at column 0
    with pytest.raises(BorderEdgeError):
        admit(GridGraph(2, 1, [0, 0], [0, 0], nb))
    with pytest.raises(ShapeError):
        GridGraph(2, 2, [0, 0], [0, 0, 0, 0], np.zeros((4, 4)))
    g = mk(2, 2, src=1)
    assert admit(g) is g and not g.src_cap.flags.writeable


def test_cut_cost_examples():
    g = mk(2, 1, src=[5, 0], snk=[0, 3], right=[2, 0], left=[0, 2])
    assert cut_cost(g, [1, 0]) == 2
    assert cut_cost(g, [0, 0]) == 5
    assert cut_cost(g, [1, 1]) == 3
    with pytest.raises(ShapeError):
        cut_cost(g, [1])
    rng = np.random.default_rng(0)
    for _ in range(30):
        w, h = int(rng.integers(1, 6)), int(rng.integers(1, 6))
        g = mk(w, h, *(rng.integers(0, 9, w * h) for _ in range(6)))
        lab = rng.integers(0, 2, w * h)
        assert cut_cost(g, lab) == oracle.cut_cost(w, h, g.src_cap, g.snk_cap, g.nbr_cap, lab)


# ------------------------------------------------------------- supergraph

def test_swap_algebra():
    g = mk(2, 1, src=[3, 0], snk=[0, 5], right=[2, 0], left=[0, 7])
    s = apply_swap(g)
    assert s.src_cap.tolist() == [0, 5] and s.snk_cap.tolist() == [3, 0]
    assert s.nbr_cap[1].tolist() == [7, 0] and s.nbr_cap[0].tolist() == [0, 2]
    rng = np.random.default_rng(21)
    for _ in range(20):
        w, h = int(rng.integers(1, 7)), int(rng.integers(1, 7))
        g = mk(w, h, *(rng.integers(0, 9, w * h) for _ in range(6)))
        assert apply_swap(apply_swap(g)).equals(g)
        o = oracle.apply_swap(w, h, g.src_cap, g.snk_cap, g.nbr_cap)
        s = apply_swap(g)
        assert np.array_equal(s.src_cap, o[0]) and np.array_equal(s.nbr_cap, o[2])


def test_swap_decision_and_balance():
    lean_sink = mk(3, 1, src=[9, 0, 0], snk=[0, 1, 1])
    assert swap_decision(lean_sink) is True
    assert swap_decision(apply_swap(lean_sink)) is False
    assert swap_decision(mk(2, 1, src=[5, 0], snk=[0, 5])) is False
    st = terminal_balance(mk(2, 2, src=[4, 0, 1, 0], snk=[1, 2, 0, 0]))
    assert (st.positive_count, st.negative_count, st.positive_sum, st.negative_sum) == (2, 1, 4, 2)


def test_join_layout_and_errors():
    a, b = mk(1, 1, src=4, snk=1), mk(1, 1, src=2, snk=7)
    comp, lay = join([a, b])
    assert (comp.width, comp.height, lay.bridge_columns) == (3, 1, (1,))
    with pytest.raises(SupergraphError):
        join([])
    with pytest.raises(SupergraphError):
        join([a], swapped=[True, False])
    with pytest.raises(SupergraphError):
        join([mk(2, 2), mk(2, 3)])
    comp, lay = join([mk(2, 2, src=1), mk(2, 3, snk=1)], pad=True)
    assert comp.height == 3 and comp.src_cap.reshape(3, 5)[2, :2].sum() == 0


def test_join_matches_reference_composites():
    """Golden composites (reference join, pad=True) rebuilt from their
    constituents' spans decode back identically."""
    for (w, h, s, t, nb, rec) in load_composites()[:10]:
        g = admit(GridGraph(w, h, s, t, nb))
        for (off, sw_w, _), (ow, oh) in zip(rec["segments"], rec["originals"]):
            assert sw_w == ow and off + ow <= w and oh <= h


def test_split_checks():
    graphs = [mk(1, 1, src=4, snk=1), mk(1, 1, src=2, snk=7)]
    comp, lay = join(graphs)
    with pytest.raises(SupergraphError):
        split(lay, CutResult(0, np.zeros(comp.n, np.uint8)), graphs)
    with pytest.raises(SupergraphError):
        split(lay, CutResult(3, np.zeros(comp.n, np.uint8)), graphs[:1])
    parts = split(lay, CutResult(3, np.array([1, 0, 0], np.uint8)), graphs)
    assert [p.flow for p in parts] == [1, 2]


def test_seed_supergraph_host_builder_matches_reference():
    for case in load_seed_supergraphs():
        W, H = case["width"], case["height"]
        probs = [SeedProblem(W, H, p["base"], p["slope"], p["sink"], p["pairwise"],
                             frozenset(p["fg"]), frozenset(p["bg"])) for p in case["problems"]]
        sched = LambdaSchedule(case["lambdas"])
        comp, lay, originals = build_seed_supergraph(probs, sched, case["mode"])
        assert comp.width == case["composite_width"]
        assert [s.swapped for s in lay.segments] == case["swapped"]
        lay2 = seed_layout(probs, sched, [lay.segments[i * len(sched)].swapped
                                          for i in range(len(probs))])
        assert lay2 == lay
        parts = split(lay, CutResult(case["composite_flow"],
                                     np.array(case["composite_labels"], np.uint8)), originals)
        assert [p.flow for p in parts] == case["flows"]
        assert [p.labels.tolist() for p in parts] == case["labels"]


# ------------------------------------------------------------- parametric

def tiny(**kw):
    pw = np.zeros((4, 2), np.int64)
    pw[1, 0] = pw[0, 1] = 1
    args = dict(width=2, height=1, unary_base=[1, 0], unary_slope=[2, 0], sink_base=[0, 4],
                pairwise=pw)
    args.update(kw)
    return SeedProblem(**args)


def test_schedule_rules():
    assert LambdaSchedule.default().mid_index == 9
    assert LambdaSchedule((5,)).mid_index == 0
    for bad in ((1, 1), (3, 2), (), (-1, 2)):
        with pytest.raises(ScheduleError):
            LambdaSchedule(bad)


def test_problem_validation():
    with pytest.raises(ProblemError):
        tiny(unary_slope=[-1, 0])
    with pytest.raises(ProblemError):
        tiny(fg_seeds={0}, bg_seeds={0})
    with pytest.raises(ProblemError):
        tiny(fg_seeds={2})


def test_instantiate_and_check_family_raise_alike():
    g = instantiate(tiny(), 3)
    assert g.src_cap.tolist() == [7, 0] and g.snk_cap.tolist() == [0, 4]
    p = tiny(fg_seeds={0}, bg_seeds={1})
    g = instantiate(p, 3)
    assert g.src_cap[0] == CAP_MAX and g.snk_cap[1] == CAP_MAX
    with pytest.raises(ScheduleError):
        instantiate(tiny(), -1)
    with pytest.raises(CapacityOverflowError):
        check_family(tiny(), (CAP_MAX,))
    with pytest.raises(CapacityOverflowError):
        check_family(tiny(), (1 << 61,))
    big = CAP_MAX // 2
    with pytest.raises(CapacityOverflowError):    # seed headroom guard
        check_family(tiny(unary_base=[big, big], unary_slope=[0, 0], sink_base=[0, big],
                          fg_seeds={0}), (0,))
    with pytest.raises(NegativeCapacityError):
        check_family(tiny(unary_base=[-1, 0]), (0,))
    pw = np.zeros((4, 2), np.int64)
    pw[0, 0] = 1
    with pytest.raises(BorderEdgeError):
        check_family(tiny(pairwise=pw), (0,))
    check_family(tiny(fg_seeds={0}, bg_seeds={1}), (1,))


def test_check_family_agrees_with_instantiate_on_random_problems():
    rng = np.random.default_rng(3)
    for _ in range(60):
        w, h = int(rng.integers(1, 5)), int(rng.integers(1, 5))
        n = w * h
        pw = rng.integers(-1, 4, (4, h, w))
        if rng.integers(0, 3):
            pw[0][:, 0] = pw[1][:, -1] = pw[2][0, :] = pw[3][-1, :] = 0
        p = SeedProblem(w, h, rng.integers(-1, 6, n) * rng.integers(1, 3),
                        rng.integers(0, 3, n), rng.integers(-1, 9, n),
                        pw.reshape(4, n), frozenset({0}), frozenset({n - 1}) if n > 1 else frozenset())
        lam = int(rng.choice([0, 1, 7, CAP_MAX // 2]))
        try:
            instantiate(p, lam)
            e1 = None
        except Exception as e:  # noqa: BLE001
            e1 = type(e)
        try:
            check_family(p, (lam,))
            e2 = None
        except Exception as e:  # noqa: BLE001
            e2 = type(e)
        assert e1 is e2


def test_check_seed_supergraph_modes():
    with pytest.raises(SupergraphError):
        check_seed_supergraph([tiny()], LambdaSchedule((1,)), "maybe")
    with pytest.raises(SupergraphError):
        check_seed_supergraph([], LambdaSchedule((1,)), "auto")


# ------------------------------------------------------------- scheduler

class FakeBackend(ThreadedBackend):
    """ThreadedBackend with an injected local solver (scheduler.py:141-142)."""


def test_run_dynamic_with_local_solver_hook():
    calls = []

    def solver(task):
        calls.append(task.id)
        return CutResult(task.id, np.zeros(1, np.uint8))

    tasks = [Task(id=i) for i in range(7)]
    workers = [WorkerHandle(0, slots=2), WorkerHandle(1)]
    backend = ThreadedBackend(local_solver=solver)
    try:
        sched, cuts = run_dynamic(tasks, workers, backend)
    finally:
        backend.close()
    assert sorted(cuts) == list(range(7)) and all(cuts[i].flow == i for i in range(7))
    assert len(sched.records) == 7


def test_run_dynamic_retries_once_then_aborts():
    def flaky(task):
        if task.id == 3:
            raise RuntimeError("boom")
        return CutResult(0, np.zeros(1, np.uint8))

    backend = ThreadedBackend(local_solver=flaky)
    try:
        with pytest.raises(BatchAborted):
            run_dynamic([Task(id=i) for i in range(5)], [WorkerHandle(0), WorkerHandle(1)], backend)
    finally:
        backend.close()


def test_gpu_backend_two_devices_dynamic_placement_and_retry():
    """GpuBackend over two (fake) devices through its solver= hook: tasks go
    FIFO to both devices; device 1 fails, is retired, and every task it had
    is retried once on device 0 (scheduler.py:253-292)."""
    import threading
    from paper_1509_06004_b200 import GpuBackend, gpu_workers
    seen = {0: [], 1: []}
    lock = threading.Lock()

    def fake(tasks, dev):
        with lock:
            seen[dev] += [t.id for t in tasks]
        if dev == 1:
            raise RuntimeError("device 1 lost")
        return [CutResult(t.id * 10 + dev, np.zeros(1, np.uint8)) for t in tasks]

    tasks = [Task(id=i) for i in range(12)]
    backend = GpuBackend(max_batch=4, solver=fake)
    try:
        sched, cuts = run_dynamic(tasks, gpu_workers([0, 1], slots=2), backend)
    finally:
        backend.close()
    assert sorted(cuts) == list(range(12))
    assert all(cuts[i].flow == 10 * i for i in range(12))          # all solved on device 0
    assert seen[1], "device 1 never received work"
    for tid in set(seen[1]):
        rec = sched.record_for(tid)
        assert rec.worker_id == 0 and rec.attempt == 2              # retried once, elsewhere
    assert all(sched.record_for(t).attempt == 1 for t in range(12) if t not in seen[1])


def test_gpu_backend_charges_a_failure_to_its_task():
    """A coalesced device batch that fails is re-solved task by task, so the
    innocent tasks complete and the abort names the task that failed twice."""
    import threading
    from paper_1509_06004_b200 import GpuBackend, gpu_workers
    gate = threading.Event()

    def fake(tasks, dev):
        gate.wait(5)   # let the queue fill so tasks coalesce
        if any(t.id == 3 for t in tasks):
            raise RuntimeError("bad task")
        return [CutResult(t.id, np.zeros(1, np.uint8)) for t in tasks]

    backend = GpuBackend(max_batch=8, solver=fake)
    threading.Timer(0.2, gate.set).start()
    try:
        with pytest.raises(BatchAborted, match="task 3 failed twice"):
            run_dynamic([Task(id=i) for i in range(6)], gpu_workers([0, 1], slots=6), backend)
    finally:
        gate.set()
        backend.close()


# ------------------------------------------------------------- synth

def test_quantize_weights_rounds_half_up():
    """harness/synth.py:139-151 semantics (test_harness.py:78-84)."""
    from paper_1509_06004_b200.synth import quantize_weights
    assert quantize_weights([0.0, 0.125, 0.375, 1.0], scale=4).tolist() == [0, 1, 2, 4]
    with pytest.raises(ValueError):
        quantize_weights([-0.1])
    with pytest.raises(ValueError):
        quantize_weights([1.0], scale=0)


def test_synth_type_b_and_lattice():
    from paper_1509_06004_b200 import synth
    b = synth.generate(24, 20, 2, 3, rng_seed=1, types=("A", "B"))
    assert len(b.problems) == 12 and b.coords == synth.lattice(24, 20, 2, 3)
    a, bb = b.problems[0], b.problems[1]
    assert a.fg_seeds == bb.fg_seeds
    top = set(range(24))
    assert bb.bg_seeds == a.bg_seeds - top
    assert np.array_equal(a.unary_base, bb.unary_base)


def test_overlap_reference_fixtures():
    """harness/bench.py:36-45 semantics (test_harness.py:119-130,
    test_acceptance.py:215-221)."""
    from fractions import Fraction
    from paper_1509_06004_b200.scoring import CutScore, overlap, scores_from_counts
    assert overlap([1, 0, 1], [1, 0, 1]) == Fraction(1)
    assert overlap([1, 1, 0, 0], [0, 0, 1, 1]) == Fraction(0)
    assert overlap([1, 1, 0, 0], [1, 1, 1, 1]) == Fraction(1, 2)
    with pytest.raises(ValueError):
        overlap([1, 0], [1, 0, 0])
    with pytest.raises(ValueError):
        overlap([0, 0], [0, 0])
    assert scores_from_counts([3], [2], [4]) == (CutScore(3, Fraction(1, 2)),)
    with pytest.raises(ValueError):
        scores_from_counts([0], [0], [0])


def test_synth_truths_match_reference():
    """Our generator reproduces the reference's problems and truth masks
    (harness/synth.py:102-136) for the scored golden batch."""
    import hashlib
    from conftest import load_scores, problem_digest
    from paper_1509_06004_b200 import synth
    g = load_scores()
    b = synth.generate(g["width"], g["height"], g["rows"], g["cols"], rng_seed=g["rng_seed"])
    assert len(b.problems) == len(g["problems"])
    for p, t, rec in zip(b.problems, b.truths, g["problems"]):
        assert problem_digest(p) == rec["problem_sha256"]
        assert hashlib.sha256(np.asarray(t, np.uint8).tobytes()).hexdigest() == rec["truth_sha256"]


def test_label_buffer_pool_never_hands_out_live_memory():
    """_native._LabelBuffers reuses a label output buffer only once no array
    (or view of one) returned earlier still references it."""
    from paper_1509_06004_b200._native import _LabelBuffers
    pool = _LabelBuffers()
    pool.MIN_BYTES = 1
    a = pool.take((2, 3, 4))
    view = a[1][2]
    del a
    b = pool.take((2, 3, 4))
    assert not np.shares_memory(b, view)      # a view of the first buffer is alive
    view[:] = 7
    del b
    c = pool.take((2, 3, 4))
    assert not np.shares_memory(c, view)
    assert (view == 7).all()
    del view
    d = pool.take((2, 3, 4))
    e = pool.take((2, 3, 4))
    assert not np.shares_memory(d, e)
    assert pool.take((5,)).shape == (5,)
