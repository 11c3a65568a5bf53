"""Single-graph max-flow / min-cut entry points (device-backed).

Mirror of /root/reference/pkg/src/pmflow/solvers.py's public surface:
``maxflow_pushrelabel(g) -> CutResult`` (solvers.py:188-191) returns the
maximum flow and the canonical minimal-source-side mask, bit-identical to
the reference; ``SolverError`` / ``NonMaximalFlowError`` are the same
exception classes (solvers.py:33-38).  The work runs on the CUDA engine
(libpmflow_b200.so); there is no CPU solver in this package.
"""

from __future__ import annotations

from .grid import CutResult, GridGraph, admit


class SolverError(RuntimeError):
    pass


class NonMaximalFlowError(SolverError):
    """The residual state does not correspond to a maximum flow."""


def maxflow_pushrelabel(g: GridGraph, device: int = 0) -> CutResult:
    """Maximum flow value plus canonical min-cut labels for an admitted graph."""
    from .supergraph import solve_composite
    return solve_composite(g, None, device=device)


def maxflow_many(graphs, device: int = 0):
    """Solve several independent graphs in one device batch (list of
    CutResult, in order)."""
    from . import _native
    graphs = list(graphs)
    for g in graphs:
        admit(g)
    items = [(g.width, g.height, g.src_cap, g.snk_cap, g.nbr_cap, None) for g in graphs]
    out = _native.solver_for_thread(device).solve_composites(items)
    return [CutResult(f, l) for f, l in out]
