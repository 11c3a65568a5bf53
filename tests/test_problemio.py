"""``.pmf`` batch files (harness/problemio.py format) against a file the
reference wrote (tests/golden/make_pmf_golden.py): read, byte-exact
rewrite, malformed files, and the problems solved on the GPU against the
oracle."""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

import oracle
from conftest import GOLDEN
from paper_1509_06004_b200 import problemio
from paper_1509_06004_b200.wire import frame

PMF = os.path.join(GOLDEN, "batch_small.pmf")


def test_reads_the_reference_file_and_rewrites_it_byte_exact(tmp_path):
    meta, probs, truths = problemio.read_problem_file(PMF)
    with open(os.path.join(GOLDEN, "batch_small.json")) as f:
        assert meta == json.load(f)
    assert len(probs) == meta["problems"] == 4 and len(truths) == 4
    assert all(p.width == 24 and p.height == 18 for p in probs)
    assert all(t.shape == (24 * 18,) and t.dtype == np.uint8 for t in truths)
    out = problemio.write_problem_file(tmp_path / "again.pmf", probs, truths,
                                       meta={k: v for k, v in meta.items()
                                             if k not in ("format", "version", "problems", "truths")})
    assert out.read_bytes() == open(PMF, "rb").read()
    assert json.loads((tmp_path / "again.json").read_text()) == meta


def _write(tmp_path, records):
    p = tmp_path / "bad.pmf"
    p.write_bytes(b"".join(frame(r) for r in records))
    return p


def test_malformed_files(tmp_path):
    raw = open(PMF, "rb").read()
    head_len = int.from_bytes(raw[:4], "little")
    header = raw[4:4 + head_len]
    second = raw[4 + head_len:]
    prob_len = int.from_bytes(second[:4], "little")
    prob = second[4:4 + prob_len]
    cases = {
        "first record is": [prob],
        "duplicate header": [header, header],
        "unknown record magic": [header, b"XXXX" + prob[4:]],
        "header promises": [header, prob],
        "problem record truncated": [header.replace(b'"problems":4', b'"problems":1'), prob[:-5]],
        "trailing bytes": [header.replace(b'"problems":4', b'"problems":1'), prob + b"\0"],
    }
    for msg, recs in cases.items():
        with pytest.raises(problemio.ProblemFileError, match=msg):
            problemio.read_problem_file(_write(tmp_path, recs))
    empty = tmp_path / "empty.pmf"
    empty.write_bytes(b"")
    with pytest.raises(problemio.ProblemFileError, match="no header"):
        problemio.read_problem_file(empty)


@pytest.mark.gpu
def test_file_problems_solved_on_gpu_match_oracle(engine):
    """The file's problems over its lambda ladder through the public seed
    supergraph API: every (problem, lambda) flow and mask equals the
    oracle's restatement of the reference solver."""
    from paper_1509_06004_b200 import LambdaSchedule, solve_seed_supergraph
    meta, probs, truths = problemio.read_problem_file(PMF)
    lams = meta["lambda_values"]
    res = solve_seed_supergraph(probs, LambdaSchedule(lams), "auto", truths=truths)
    K = len(lams)
    for pi, p in enumerate(probs):
        for j, lam in enumerate(lams):
            src, snk, nbr = oracle.instantiate(p.unary_base, p.unary_slope, p.sink_base, p.pairwise,
                                               p.fg_seeds, p.bg_seeds, lam)
            f, lab, _ = oracle.solve(p.width, p.height, src, snk, nbr)
            cut = res.cuts[pi * K + j]
            assert cut.flow == f
            assert np.array_equal(np.asarray(cut.labels, np.uint8).reshape(-1), lab)


def test_writer_rejects_mismatched_truths(tmp_path):
    meta, probs, truths = problemio.read_problem_file(PMF)
    with pytest.raises(problemio.ProblemFileError, match="one truth mask per problem"):
        problemio.write_problem_file(tmp_path / "x.pmf", probs, truths[:-1])
    # no truths at all is fine, and reads back with an empty list
    problemio.write_problem_file(tmp_path / "y.pmf", probs)
    m2, p2, t2 = problemio.read_problem_file(tmp_path / "y.pmf")
    assert t2 == [] and m2["truths"] == 0 and len(p2) == len(probs)
    assert all(np.array_equal(a.pairwise, b.pairwise) and a.fg_seeds == b.fg_seeds
               for a, b in zip(p2, probs))
