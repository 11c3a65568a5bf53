"""Host side of on-device synthesis (synth_device.py): the images are the
reference generator's, the histogram statistics equal the materialised
problems' (so admission raises what the host problems raise, in order), and
the stand-in problems rebuild the host planes exactly.  Device planes and
cuts: tests/test_gpu_synth.py."""

from __future__ import annotations

import numpy as np
import pytest

from paper_1509_06004_b200 import CapacityOverflowError, LambdaSchedule, synth
from paper_1509_06004_b200 import synth_device as sd
from paper_1509_06004_b200.supergraph import check_seed_supergraph


def _host(W, H, r, c, seeds, types):
    out = []
    for s in seeds:
        out += synth.generate(W, H, r, c, rng_seed=s, types=types).problems
    return out


@pytest.mark.parametrize("shape", [(40, 30, 2, 2), (7, 5, 1, 1), (3, 3, 1, 1), (64, 9, 1, 3)])
def test_family_stats_equal_materialised_problems(shape):
    W, H, r, c = shape
    seeds = (0, 1, 5)
    b = sd.generate_images(W, H, r, c, rng_seeds=seeds, types=("A", "B"))
    host = _host(W, H, r, c, seeds, ("A", "B"))
    for i, s in enumerate(seeds):
        assert np.array_equal(b.images[i], synth.generate(W, H, r, c, rng_seed=s).image)
    fams = b.families()
    assert len(fams) == len(host)
    for f, p in zip(fams, host):
        assert f._family_stats() == p._family_stats()
        q = f.problem()
        for name in ("unary_base", "unary_slope", "sink_base", "pairwise"):
            assert np.array_equal(getattr(q, name), getattr(p, name)), name
        assert q.fg_seeds == p.fg_seeds and q.bg_seeds == p.bg_seeds
    truths = synth.generate(W, H, r, c, rng_seed=5, types=("A", "B")).truths
    assert all(np.array_equal(a, t) for a, t in zip(b.truths[-len(truths):], truths))


@pytest.mark.parametrize("lams", [(1, 3, 9), (2, 600), (1, 5000), (1, 10 ** 6), (1, 3, 1 << 27)])
def test_admission_errors_match_host_problems(lams):
    """Same exception class and message as check_seed_supergraph on the
    host-built problems, including the exact fallbacks near CAP_MAX."""
    sched = LambdaSchedule(lams)
    b = sd.generate_images(48, 36, 2, 2, rng_seeds=(3, 4), types=("A", "B"))
    host = _host(48, 36, 2, 2, (3, 4), ("A", "B"))
    for mode in ("auto", "on"):
        want = got = None
        try:
            check_seed_supergraph(host, sched, mode)
        except Exception as exc:  # noqa: BLE001
            want = (type(exc), str(exc))
        try:
            check_seed_supergraph(b.families(), sched, mode)
        except Exception as exc:  # noqa: BLE001
            got = (type(exc), str(exc))
        assert got == want


def test_overflow_is_raised():
    b = sd.generate_images(48, 36, 1, 1, rng_seeds=(0,))
    with pytest.raises(CapacityOverflowError):
        check_seed_supergraph(b.families(), LambdaSchedule((1, 10 ** 6)))


def test_image_batch_validation():
    with pytest.raises(ValueError):
        sd.ImageBatch(np.zeros((4, 4)), [(1, 1)])
    with pytest.raises(ValueError):
        sd.ImageBatch(np.full((1, 4, 4), 256), [(1, 1)])
    with pytest.raises(ValueError):
        sd.ImageBatch(np.zeros((1, 4, 4)), [(1, 1)], types=("C",))
    with pytest.raises(ValueError, match="border"):
        sd.ImageBatch(np.zeros((1, 4, 4), np.uint8), [(0, 1)]).families()
    # type B: the top row is not background
    assert len(sd.ImageBatch(np.zeros((1, 4, 4), np.uint8), [(1, 0)], types=("B",)).families()) == 1


def test_admission_order_across_images_and_types():
    """The first failing (image, seed, type) problem decides the error, as
    check_seed_supergraph on the host problems in the same order."""
    sched = LambdaSchedule((1, 700, 140000))
    b = sd.generate_images(64, 48, 2, 2, rng_seeds=(5, 6, 7), types=("B", "A"))
    host = []
    for s in (5, 6, 7):
        host += synth.generate(64, 48, 2, 2, rng_seed=s, types=("B", "A")).problems
    outcome = []
    for probs in (host, b.families()):
        try:
            check_seed_supergraph(probs, sched, "auto")
            outcome.append(None)
        except Exception as exc:  # noqa: BLE001
            outcome.append((type(exc), str(exc)))
    assert outcome[0] == outcome[1]


def test_tiny_images():
    """3x3 images: one interior pixel, the seed; the border is background
    (type A) or the ring minus its top row (type B)."""
    b = sd.ImageBatch(np.array([[[0, 9, 2], [3, 40, 5], [6, 7, 255]]], np.uint8), [(1, 1)], ("A", "B"))
    fa, fb = b.families()
    assert fa.n == 9 and len(fa.bg_seeds) == 8 and len(fb.bg_seeds) == 5
    for f in (fa, fb):
        p = f.problem()
        assert f._family_stats() == p._family_stats()
