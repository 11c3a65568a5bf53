"""paper_1509_06004_b200 -- B200-native parametric max-flow engine for the
supergraph framework of arXiv 1509.06004 (reference package ``pmflow``).

Drop-in names for the reference's hot path (/root/reference/pkg/src/pmflow/
__init__.py:4-32, the in-scope subset): graph core, lambda schedules and
seed problems, supergraph knitting, ``solve_composite`` and the dynamic
scheduler.  Solves run on hand-written sm_100a CUDA kernels
(libpmflow_b200.so, C ABI in include/pmflow_b200.h); there is no CPU
fallback.
"""

from .floatcap import FloatCutResult, maxflow_float, maxflow_float_many, quantize_graph
from .grid import (CAP_MAX, BorderEdgeError, CapacityOverflowError, CutResult, GraphError,
                   GridGraph, NegativeCapacityError, ShapeError, admit, cut_cost)
from .parametric import (DEFAULT_LAMBDA_VALUES, HALVED_LAMBDA_VALUES, LambdaSchedule,
                         ParametricResult, ProblemError, ScheduleError, SeedProblem,
                         check_nested, energy, instantiate, solve_schedule_sequential)
from .scheduler import (BatchAborted, GpuBackend, SchedulerError, Task, TaskSchedule,
                        ThreadedBackend, WorkerFailure, WorkerHandle, gpu_workers, run_dynamic)
from .solvers import NonMaximalFlowError, SolverError, maxflow_many, maxflow_pushrelabel
from .supergraph import (SeedSupergraphResult, Segment, SupergraphError, SupergraphLayout,
                         apply_swap, build_lambda_supergraph, build_seed_supergraph,
                         family_swap_decision, join, solve_composite, solve_composites,
                         solve_seed_supergraph, solve_seed_supergraphs, split, swap_decision,
                         terminal_balance)

__version__ = "0.1.0"

__all__ = [
    "CAP_MAX", "BatchAborted", "FloatCutResult", "maxflow_float", "maxflow_float_many", "quantize_graph", "BorderEdgeError", "CapacityOverflowError", "CutResult",
    "DEFAULT_LAMBDA_VALUES", "GpuBackend", "GraphError", "GridGraph", "HALVED_LAMBDA_VALUES",
    "LambdaSchedule", "NegativeCapacityError", "NonMaximalFlowError", "ParametricResult",
    "ProblemError", "ScheduleError", "SchedulerError", "SeedProblem", "SeedSupergraphResult",
    "Segment", "ShapeError", "SolverError", "SupergraphError", "SupergraphLayout", "Task",
    "TaskSchedule", "ThreadedBackend", "WorkerFailure", "WorkerHandle", "admit", "apply_swap",
    "build_lambda_supergraph", "build_seed_supergraph", "check_nested", "cut_cost", "energy",
    "family_swap_decision", "gpu_workers", "instantiate", "join", "maxflow_many",
    "maxflow_pushrelabel", "run_dynamic", "solve_composite", "solve_composites",
    "solve_schedule_sequential", "solve_seed_supergraph", "solve_seed_supergraphs", "split", "swap_decision",
    "terminal_balance", "__version__",
]
