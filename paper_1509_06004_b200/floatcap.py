"""Float-capacity mode: real-valued grid graphs solved on the integer engine.

The reference has no float solver; real-valued weights enter it only
through ``quantize_weights`` (harness/synth.py:139-151: round half up at
``scale``, default 2**16, negatives rejected) and then run the integer path.
This module does the same in one call: quantise every capacity plane at
``scale`` (``inf`` -> CAP_MAX, the hard-constraint value seeds use,
parametric.py:150-153), admit the graph (grid.py:102-130), solve it on the
GPU (either state variant), and rescale the flow by ``1 / scale``.

Accuracy: every capacity moves by at most 0.5 / scale, so a cut of k finite
arcs moves by at most k / (2 scale); the flow is within 1e-5 relative error
of the fp64 maximum flow for weights of order one and above (tested against
an fp64 max-flow, tests/test_gpu_float.py).  Labels are the minimal source
side of the QUANTISED graph; pixels where it differs from the fp64 minimal
source side are ties (cuts within the quantisation error of each other) and
are reported by ``label_report``, not hidden.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .grid import CAP_MAX, CapacityOverflowError, GridGraph, admit
from .synth import quantize_weights

FLOAT_SCALE = 1 << 16


@dataclass(frozen=True, eq=False)
class FloatCutResult:
    flow: float            # int_flow / scale
    labels: np.ndarray     # uint8 (n,), 1 = source side of the quantised graph
    int_flow: int          # flow of the quantised graph
    scale: int


def _plane(values, count, scale, label):
    a = np.asarray(values, np.float64).reshape(-1)
    if a.size != count:
        raise ValueError(f"{label}: expected {count} entries, got {a.size}")
    if np.isnan(a).any():
        raise ValueError(f"{label}: NaN capacity")
    inf = np.isposinf(a)
    q = quantize_weights(np.where(inf, 0.0, a), scale)
    if q.size and int(q.max()) > CAP_MAX:
        raise CapacityOverflowError(f"{label}: a capacity times scale {scale} exceeds CAP_MAX = 2**30")
    q[inf] = CAP_MAX
    return q


def quantize_graph(width: int, height: int, src, snk, nbr, scale: int = FLOAT_SCALE) -> GridGraph:
    """Admitted integer GridGraph of float capacities (quantize_weights per
    plane; +inf -> CAP_MAX)."""
    n = width * height
    g = GridGraph(width, height, _plane(src, n, scale, "src_cap"), _plane(snk, n, scale, "snk_cap"),
                  _plane(nbr, 4 * n, scale, "nbr_cap").reshape(4, n))
    return admit(g)


def maxflow_float_many(graphs, scale: int = FLOAT_SCALE, device: int = 0):
    """graphs: [(width, height, src, snk, nbr)] float planes -> [FloatCutResult],
    all solved in one device batch."""
    from .supergraph import solve_composites
    qs = [quantize_graph(w, h, s, t, nb, scale) for (w, h, s, t, nb) in graphs]
    cuts = solve_composites([(g, None) for g in qs], device=device)
    return [FloatCutResult(c.flow / scale, np.asarray(c.labels, np.uint8), int(c.flow), scale) for c in cuts]


def maxflow_float(width, height, src, snk, nbr, scale: int = FLOAT_SCALE, device: int = 0) -> FloatCutResult:
    """One float-capacity graph (maxflow_pushrelabel, solvers.py:188-191,
    behind quantize_weights)."""
    return maxflow_float_many([(width, height, src, snk, nbr)], scale, device)[0]


def cut_cost_float(width, height, src, snk, nbr, labels) -> float:
    """fp64 cost of the cut given by a 0/1 mask (grid.py:159-178 semantics)."""
    lab = np.asarray(labels, bool).reshape(height, width)
    src = np.asarray(src, np.float64).reshape(height, width)
    snk = np.asarray(snk, np.float64).reshape(height, width)
    nb = np.asarray(nbr, np.float64).reshape(4, height, width)
    cost = float(snk[lab].sum() + src[~lab].sum())
    pad = np.ones((height + 2, width + 2), bool)
    pad[1:-1, 1:-1] = lab
    nb_lab = (pad[1:-1, :-2], pad[1:-1, 2:], pad[:-2, 1:-1], pad[2:, 1:-1])
    for d in range(4):
        cost += float(nb[d][lab & ~nb_lab[d]].sum())
    return cost


def label_report(res: FloatCutResult, ref_labels, width, height, src, snk, nbr) -> dict:
    """Tie-pixel report of a float solve against reference labels (e.g. an
    fp64 solver's minimal source side): how many pixels differ, and the fp64
    cost of both cuts -- differing pixels are ties when the two costs agree
    within the quantisation error."""
    ref = np.asarray(ref_labels, np.uint8).reshape(-1)
    diff = int(np.count_nonzero(res.labels != ref))
    c_res = cut_cost_float(width, height, src, snk, nbr, res.labels)
    c_ref = cut_cost_float(width, height, src, snk, nbr, ref)
    return {"mismatched_pixels": diff, "cost": c_res, "reference_cost": c_ref,
            "cost_rel_gap": abs(c_res - c_ref) / max(abs(c_ref), 1e-300)}
