"""On-device synthesis (pmf_synth_stage, synth_device.py) against the host
generator: the planes the GPU derives equal synth.generate's planes
element for element, and every cut, layout and score equals what
solve_seed_supergraph returns for the host-built problems (which
test_gpu_parity.py pins to the reference and the oracle)."""

from __future__ import annotations

import numpy as np
import pytest

from paper_1509_06004_b200 import (LambdaSchedule, _native, solve_seed_supergraph, solve_seed_supergraphs,
                                   synth)
from paper_1509_06004_b200 import synth_device as sd

pytestmark = pytest.mark.gpu


def _host(W, H, r, c, seeds, types):
    out = []
    for s in seeds:
        out += synth.generate(W, H, r, c, rng_seed=s, types=types).problems
    return out


def _same(a, b):
    assert a.layout == b.layout
    assert [c.flow for c in a.cuts] == [c.flow for c in b.cuts]
    assert all(np.array_equal(x.labels, y.labels) for x, y in zip(a.cuts, b.cuts))
    assert a.scores == b.scores


def test_device_planes_equal_host_planes():
    W, H = 53, 37   # odd sizes: partial tiles, ragged 4-pixel groups
    seeds = (0, 7, 11)
    b = sd.generate_images(W, H, 2, 3, rng_seeds=seeds, types=("A", "B"))
    s = _native.solver_for_thread(0)
    s.synth_stage(b.images, b.coords, b.types, (1, 2, 3), "auto")
    s.seed_run()
    pl, pw = s.debug_planes()
    n = W * H
    host = _host(W, H, 2, 3, seeds, ("A", "B"))
    nseed = len(b.coords)
    for i in range(len(seeds)):
        for k in range(nseed):
            p = host[(i * nseed + k) * 2]
            u = i * nseed + k
            for j, name in enumerate(("unary_base", "unary_slope", "sink_base")):
                assert np.array_equal(pl[(3 * u + j) * n:(3 * u + j + 1) * n], getattr(p, name)), (i, k, name)
        assert np.array_equal(pw[4 * i * n:4 * (i + 1) * n].reshape(4, n), host[i * nseed * 2].pairwise)


@pytest.mark.parametrize("cfg", [(160, 120, 2, 2, (0, 1, 2), ("A", "B")), (96, 64, 1, 3, (5,), ("A",)),
                                 (120, 90, 2, 1, (3, 4), ("B",))])
def test_cuts_equal_host_problem_path(cfg):
    W, H, r, c, seeds, types = cfg
    sched = LambdaSchedule(synth.L20[:8])
    b = sd.generate_images(W, H, r, c, rng_seeds=seeds, types=types)
    want = solve_seed_supergraph(_host(W, H, r, c, seeds, types), sched, "auto", truths=b.truths)
    got = sd.solve_image_batch(b, sched, "auto", truths=b.truths)
    _same(got, want)
    for mode in ("on", "off"):
        _same(sd.solve_image_batch(b, sched, mode), solve_seed_supergraph(b.problems(), sched, mode))


def test_cpmc_image_equals_host_path():
    """One C3 image (25 seeds x 2 types x L20), planes built on the device."""
    sched = LambdaSchedule(synth.L20)
    b = sd.generate_images(500, 375, 5, 5, rng_seeds=(17,), types=("A", "B"))
    want = solve_seed_supergraph(synth.generate(500, 375, 5, 5, rng_seed=17, types=("A", "B")).problems, sched)
    _same(sd.solve_image_batch(b, sched), want)


def test_stream_mixes_image_batches_and_problem_lists():
    sched = LambdaSchedule(synth.L20[:6])
    b0 = sd.generate_images(160, 120, 2, 2, rng_seeds=(0, 1), types=("A", "B"))
    p1 = _host(160, 120, 2, 2, (2,), ("A", "B"))
    b2 = sd.generate_images(160, 120, 2, 2, rng_seeds=(3,), types=("A", "B"))
    want = [solve_seed_supergraph(b0.problems(), sched), solve_seed_supergraph(p1, sched),
            solve_seed_supergraph(b2.problems(), sched)]
    got = list(solve_seed_supergraphs([b0, p1, b2], sched))
    for g, w in zip(got, want):
        _same(g, w)


def test_synth_stage_rejects_bad_arguments():
    s = _native.solver_for_thread(0)
    img = np.zeros((1, 8, 8), np.uint8)
    with pytest.raises(ValueError):
        s.synth_stage(img, [(0, 3)], ("A",), (1, 2))          # seed on the border
    with pytest.raises(ValueError):
        s.synth_stage(img, [(3, 9)], ("A",), (1, 2))          # outside the image
    with pytest.raises(ValueError):
        s.synth_stage(img, [(3, 3)], ("A",), (2, 1))          # lambdas not increasing
    s.synth_stage(img, [(3, 0)], ("B",), (1, 2))              # type B: the top row is not background


def test_synthetic_batch_on_the_int64_state_variant():
    """force_wide: the int64 state variant (wide.cuh) reads the device-built
    planes exactly like staged ones."""
    sched = LambdaSchedule(synth.L20[:5])
    b = sd.generate_images(96, 64, 2, 1, rng_seeds=(8,), types=("A", "B"))
    want = sd.solve_image_batch(b, sched)
    s = _native.solver_for_thread(0)
    s.set("force_wide", 1)
    try:
        got = sd.solve_image_batch(b, sched)
        assert s.stats()["wide_mode"] == 1
    finally:
        s.set("force_wide", 0)
    _same(got, want)


def test_launch_wait_contract():
    """pmf_seed_launch / pmf_seed_wait: launch behind another solver's run,
    wait reports the run; misuse is an argument error, not a hang."""
    sched = LambdaSchedule(synth.L20[:4])
    probs = synth.generate(96, 64, 1, 2, rng_seed=3).problems
    a, b = _native.Solver(0), _native.Solver(0)
    try:
        with pytest.raises(ValueError):
            a.seed_wait()                          # nothing launched
        with pytest.raises(ValueError):
            a.seed_launch()                        # nothing staged
        a.seed_stage(96, 64, probs, sched.values)
        b.seed_stage(96, 64, probs[::-1], sched.values)
        with pytest.raises(ValueError):
            a.seed_launch(a)                       # cannot wait for itself
        a.seed_launch()
        b.seed_launch(a)                           # runs after a's run
        b.seed_wait()
        a.seed_wait()
        _, fa, _ = a.seed_fetch(False)
        _, fb, _ = b.seed_fetch(False)
        assert np.array_equal(fa, fb[::-1])
        want = solve_seed_supergraph(probs, sched)
        assert [c.flow for c in want.cuts] == [int(f) for f in fa.reshape(-1)]
    finally:
        a.close()
        b.close()


def test_nested_streams_use_separate_solvers():
    """A stream consumed inside another stream's loop (same thread) leases
    its own solvers: both yield what the single calls return."""
    sched = LambdaSchedule(synth.L20[:4])
    outer = [_host(96, 64, 1, 2, (s,), ("A",)) for s in (1, 2)]
    inner = [sd.generate_images(96, 64, 1, 2, rng_seeds=(s,)) for s in (3, 4)]
    want_o = [solve_seed_supergraph(b, sched) for b in outer]
    want_i = [sd.solve_image_batch(b, sched) for b in inner]
    for k, ro in enumerate(solve_seed_supergraphs(outer, sched)):
        _same(ro, want_o[k])
        for j, ri in enumerate(solve_seed_supergraphs(inner, sched)):
            _same(ri, want_i[j])


def test_overlapping_async_runs_in_a_stream():
    """Consecutive asynchronous runs share the device (overlap_us: idle CTAs
    of a run's tail leave their SM to the next run; 1 us = aggressive
    yielding): every batch still equals its single call, and overlap off
    gives the same results."""
    sched = LambdaSchedule(synth.L20[:8])
    batches = [_host(160, 120, 1, 2, (s,), ("A", "B")) for s in range(10)]
    want = [solve_seed_supergraph(b, sched) for b in batches]
    for ov in (1, 20, 0):
        for g, w in zip(solve_seed_supergraphs(batches, sched, overlap_us=ov), want):
            _same(g, w)
