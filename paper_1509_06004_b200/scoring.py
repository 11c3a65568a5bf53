"""Scoring of decoded cuts against ground truth (harness/bench.py).

``overlap`` is the reference's exact Jaccard overlap on the host
(harness/bench.py:36-45, same errors and Fraction result).  ``score_cuts``
computes the same numbers -- and the per-cut foreground counts of
harness/bench.py:104-111 -- for a whole device batch on the GPU, from the
label planes still resident after the solve (``pmf_seed_score``), instead
of a host loop over every (seed, lambda) mask.
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

import numpy as np


def overlap(mask, truth) -> Fraction:
    """Exact Jaccard overlap |S & G| / |S | G| of two 0/1 masks."""
    a = np.asarray(mask).reshape(-1).astype(bool)
    b = np.asarray(truth).reshape(-1).astype(bool)
    if a.size != b.size:
        raise ValueError(f"mask sizes differ: {a.size} vs {b.size}")
    union = int((a | b).sum())
    if union == 0:
        raise ValueError("overlap of two empty masks is undefined")
    return Fraction(int((a & b).sum()), union)


@dataclass(frozen=True)
class CutScore:
    """Foreground pixel count and exact overlap of one decoded cut."""

    foreground: int
    overlap: Fraction


def scores_from_counts(fg, inter, union) -> tuple:
    """CutScore per (problem, lambda), problem-major, from device counts."""
    out = []
    for f, i, u in zip(np.asarray(fg).reshape(-1), np.asarray(inter).reshape(-1),
                       np.asarray(union).reshape(-1)):
        if int(u) == 0:
            raise ValueError("overlap of two empty masks is undefined")
        out.append(CutScore(int(f), Fraction(int(i), int(u))))
    return tuple(out)


def score_cuts(solver, truths) -> tuple:
    """Device scores of the solver's last seed batch: one truth mask per
    problem; CutScore per (problem, lambda), problem-major."""
    return scores_from_counts(*solver.seed_score(truths))
