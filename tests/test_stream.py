"""Host logic of the batch stream (supergraph.solve_seed_supergraphs) with a
fake engine: ordering, error placement, serialised device runs and the
overlap of staging with the previous batch's run.  The GPU parity of the
stream against solve_seed_supergraph is in test_gpu_parity.py."""

from __future__ import annotations

import threading
import time

import numpy as np
import pytest

from paper_1509_06004_b200 import CapacityOverflowError, LambdaSchedule, _native, synth
from paper_1509_06004_b200 import supergraph as sg


class FakeSolver:
    """seed_stage / seed_launch / seed_wait / seed_fetch with the engine's
    call contract on a simulated device timeline (a launched run starts when
    `after`'s run has ended); flows encode (batch tag, problem, lambda)."""

    log = []
    RUN_S = 0.15

    def __init__(self, slot):
        self.slot = slot
        self.staged = None
        self.end = 0.0
        self.deps = []

    def seed_stage(self, W, H, problems, lambdas, swap_mode):
        FakeSolver.log.append(("stage", problems[0].tag, time.perf_counter(), None))
        self.staged = (W * H, problems, len(lambdas))

    def set(self, name, value):
        pass

    def seed_kind(self):
        return False, False   # step-synchronous runs: never share the device

    def depend(self, other):
        self.deps.append(other)

    def seed_launch(self, after=None):
        deps = self.deps + ([after] if after is not None else [])
        self.deps = []
        start = max([time.perf_counter()] + [d.end for d in deps])
        self.end = start + FakeSolver.RUN_S
        FakeSolver.log.append(("run", self.staged[1][0].tag, start, self.end))

    def seed_wait(self):
        time.sleep(max(0.0, self.end - time.perf_counter()))

    def abandon(self):
        pass

    def seed_fetch(self, labels=True):
        n, probs, K = self.staged
        tag = probs[0].tag
        flows = np.array([[tag * 1000 + 10 * i + j for j in range(K)] for i in range(len(probs))], np.int64)
        lab = np.zeros((len(probs), K, n), np.uint8)
        return np.zeros(len(probs), bool), flows, lab


def _batch(tag):
    b = synth.generate(24, 16, 1, 2, rng_seed=tag, types=("A",))
    probs = list(b.problems)
    for p in probs:
        object.__setattr__(p, "tag", tag)   # frozen dataclass: a trace tag for the fake engine
    return probs


@pytest.fixture
def fake_engine(monkeypatch):
    FakeSolver.log = []
    solvers = [FakeSolver(i) for i in range(4)]
    monkeypatch.setattr(_native, "pipeline_solvers", lambda device, depth, lease=False: solvers[:depth])
    monkeypatch.setattr(_native, "release_solvers", lambda device, s: None)
    return solvers


def test_stream_order_overlap_and_serial_runs(fake_engine):
    sched = LambdaSchedule((1, 3, 9))
    batches = [_batch(t) for t in range(4)]
    out = list(sg.solve_seed_supergraphs(batches, sched))
    assert [r.cuts[0].flow // 1000 for r in out] == [0, 1, 2, 3]
    for t, r in enumerate(out):
        assert [c.flow for c in r.cuts] == [t * 1000 + 10 * i + j for i in range(2) for j in range(3)]
        assert len(r.layout.segments) == 6
    runs = sorted((t, a, b) for k, t, a, b in FakeSolver.log if k == "run")
    assert [t for t, _, _ in runs] == [0, 1, 2, 3]
    for (_, _, e0), (_, s1, _) in zip(runs, runs[1:]):
        assert s1 >= e0                          # device runs never overlap
    stage = {t: a for k, t, a, _ in FakeSolver.log if k == "stage"}
    # batch k + 1 was staged while batch k was running
    assert all(stage[t + 1] < runs[t][2] for t in range(3))


def test_stream_raises_at_the_failing_batch(fake_engine):
    sched = LambdaSchedule((1, 3, 9))
    good = [_batch(t) for t in range(3)]
    bad = _batch(7)
    huge = LambdaSchedule((1, 3, 1 << 29))   # instantiate overflows CAP_MAX at the top lambda
    with pytest.raises(CapacityOverflowError):
        sg.check_seed_supergraph(bad, huge)
    # same error class, same position, through the stream (earlier results delivered first)
    gen = sg.solve_seed_supergraphs([good[0], good[1]], huge)
    with pytest.raises(CapacityOverflowError):
        next(gen)
    got = []
    with pytest.raises(sg.SupergraphError):
        for r in sg.solve_seed_supergraphs([good[0], [], good[2]], sched):
            got.append(r)
    assert [r.cuts[0].flow // 1000 for r in got] == [0]


def test_stream_closed_early_stops_its_threads(fake_engine):
    sched = LambdaSchedule((1, 3))
    before = threading.active_count()
    gen = sg.solve_seed_supergraphs((_batch(t) for t in range(6)), sched, depth=2)
    first = next(gen)
    assert first.cuts[0].flow == 0
    gen.close()
    time.sleep(0.05)
    assert threading.active_count() <= before
