"""The CPU oracle (oracle/) pinned against vectors produced by the
reference itself (tests/golden/, tests/golden/make_golden.py)."""

import numpy as np
import pytest

import oracle
from conftest import load_composites, load_kat, load_random, load_seed_supergraphs, load_synth, \
    problem_digest


def test_kat_fixtures():
    for name, k in load_kat().items():
        f, lab, _ = oracle.solve(k["width"], k["height"], k["src"], k["snk"], k["nbr"])
        assert f == k["flow"], name
        assert lab.tolist() == k["labels"], name


@pytest.mark.parametrize("name", ["random_8x8_seed101.npz", "random_3x3_seed102.npz"])
def test_random_sweeps(name):
    for (w, h, s, t, nb, flow, labels) in load_random(name):
        f, lab, _ = oracle.solve(w, h, s, t, nb)
        assert f == flow
        assert np.array_equal(lab, labels)


def test_composites_with_swapped_spans():
    for (w, h, s, t, nb, rec) in load_composites():
        segs = [tuple(x) for x in rec["segments"]]
        f, lab, _ = oracle.solve(w, h, s, t, nb, segs)
        assert f == rec["flow"]
        assert lab.tolist() == rec["labels"]


def test_seed_supergraph_builder_and_split():
    for case in load_seed_supergraphs():
        W, H = case["width"], case["height"]
        probs = [(W, H, np.array(p["base"]), np.array(p["slope"]), np.array(p["sink"]),
                  np.array(p["pairwise"]), frozenset(p["fg"]), frozenset(p["bg"]))
                 for p in case["problems"]]
        tw, h, src, snk, nbr, segs, origs = oracle.build_seed_supergraph(
            probs, case["lambdas"], case["mode"])
        assert tw == case["composite_width"]
        assert [s[2] for s in segs] == case["swapped"]
        f, lab, _ = oracle.solve(tw, h, src, snk, nbr, segs)
        assert f == case["composite_flow"]
        assert lab.tolist() == case["composite_labels"]
        parts = oracle.split(tw, h, lab, segs, origs)
        assert [p[0] for p in parts] == case["flows"]
        assert [p[1].tolist() for p in parts] == case["labels"]


def test_c1_pulse_schedule_and_flows():
    """C1 (160x120, DEFAULT ladder): per-lambda flows/labels from the
    reference, composite flow 27,814,225 and the reference's 513 pulses at
    lambda=1."""
    g = load_synth("c1_160x120.npz")
    probs = oracle.synth_problems(160, 120, 1, 1)
    assert g["composite_flow"] == 27814225
    for lam, flow, labels in zip(g["lambdas"], g["flows"], g["labels"]):
        s, t, nb = oracle.instantiate(*probs[0][2:], lam)
        f, lab, pulses = oracle.solve(160, 120, s, t, nb)
        assert f == flow and np.array_equal(lab, labels)
        if lam == 1:
            assert pulses == 513


def test_synth_restatement_matches_reference_generator():
    from paper_1509_06004_b200 import synth
    g = load_synth("c1_160x120.npz")
    batch = synth.generate(160, 120, 1, 1, rng_seed=0)
    assert problem_digest(batch.problems[0]) == g["sha"]
    o = oracle.synth_problems(160, 120, 1, 1)[0]
    p = batch.problems[0]
    for a, b in zip((p.unary_base, p.unary_slope, p.sink_base, p.pairwise), o[2:6]):
        assert np.array_equal(a, b)


def test_c2_generator_digest():
    import os
    from conftest import GOLDEN
    from paper_1509_06004_b200 import synth
    if not os.path.exists(os.path.join(GOLDEN, "c2_500x375.npz")):
        pytest.skip("C2 fixture not generated")
    g = load_synth("c2_500x375.npz")
    assert problem_digest(synth.generate(500, 375, rng_seed=0).problems[0]) == g["sha"]
    assert sum(g["flows"]) == 90475333


def test_fp64_checker_pinned_on_integer_vectors():
    """The fp64 Dinic checker of the float mode (oracle/maxflow_f64.c)
    reproduces the reference's flows and minimal source sides exactly on
    integer-valued graphs (integers are exact in double): the KATs, the 500
    random 8x8 grids and the C1 per-lambda cuts."""
    for name, k in load_kat().items():
        f, lab = oracle.maxflow_f64(k["width"], k["height"], k["src"], k["snk"], k["nbr"])
        assert f == k["flow"], name
        assert lab.tolist() == k["labels"], name
    for (w, h, s, t, nb, flow, labels) in load_random("random_8x8_seed101.npz"):
        f, lab = oracle.maxflow_f64(w, h, s, t, nb)
        assert f == flow and np.array_equal(lab, labels)
    gold = load_synth("c1_160x120.npz")
    p = oracle.synth_problems(160, 120, 1, 1, rng_seed=0)[0]
    for k in (0, 4, 19):
        src, snk, nbr = oracle.instantiate(*p[2:], gold["lambdas"][k])
        f, lab = oracle.maxflow_f64(160, 120, src, snk, nbr)
        assert f == gold["flows"][k] and np.array_equal(lab, gold["labels"][k])
