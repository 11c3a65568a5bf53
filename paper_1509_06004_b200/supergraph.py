"""Supergraphs: many grid problems knitted into one composite, solved on
the device.

Mirror of /root/reference/pkg/src/pmflow/supergraph.py.  Host helpers keep
the reference's names and semantics -- ``Segment`` / ``SupergraphLayout``
(:39-64), ``terminal_balance`` / ``swap_decision`` (:77-92), ``apply_swap``
(:95-109), ``join`` (:112-154), ``split`` (:157-187),
``family_swap_decision`` (:210-212), ``build_lambda_supergraph`` (:215-224),
``build_seed_supergraph`` (:227-253) -- and ``solve_composite`` (:190-207),
the single solver entry point, runs on the CUDA engine.

``solve_seed_supergraph`` is the fused device path: it takes the seed
problems themselves, builds every (problem, lambda) graph on the GPU (no
host composite), solves them in one batch and returns the layout plus the
per-constituent cuts -- exactly what
``split(layout, solve_composite(*build_seed_supergraph(...)[:2]), originals)``
returns, bit for bit.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass

import numpy as np

from .grid import CutResult, GridGraph, admit, cut_cost
from .parametric import prefetch_family_stats, LambdaSchedule, SeedProblem, check_family, instantiate


class SupergraphError(ValueError):
    pass


@dataclass(frozen=True)
class Segment:
    """A constituent's column span inside a composite."""

    constituent: int
    offset: int
    width: int
    swapped: bool


@dataclass(frozen=True)
class SupergraphLayout:
    """Column spans, bridge columns and height of a composite."""

    segments: tuple
    bridge_columns: tuple
    height: int

    @property
    def total_width(self) -> int:
        tail = self.segments[-1]
        return tail.offset + tail.width

    @property
    def any_swapped(self) -> bool:
        return any(s.swapped for s in self.segments)


@dataclass(frozen=True)
class SwapStats:
    """Sign pattern of src_cap - snk_cap over a graph's pixels."""

    positive_count: int
    negative_count: int
    positive_sum: int
    negative_sum: int  # absolute value


def terminal_balance(g: GridGraph) -> SwapStats:
    diff = g.src_cap - g.snk_cap
    up, down = diff[diff > 0], diff[diff < 0]
    return SwapStats(int(up.size), int(down.size), int(up.sum()), int(-down.sum()))


def swap_decision(g: GridGraph) -> bool:
    """Swap iff strictly more pixels lean to the sink than to the source."""
    st = terminal_balance(g)
    return st.negative_count > st.positive_count


def apply_swap(g: GridGraph) -> GridGraph:
    """Exchange the terminals and reverse every neighbour arc (involution).

    The arc p -> right neighbour of the swapped graph carries the original
    right-neighbour -> p capacity, i.e. the LEFT plane shifted one column,
    and likewise for the other three directions."""
    H, W = g.height, g.width
    src = g.nbr_cap.reshape(4, H, W)
    dst = np.zeros_like(src)
    dst[0][:, 1:] = src[1][:, :-1]     # L'(y, x) = R(y, x-1)
    dst[1][:, :-1] = src[0][:, 1:]     # R'(y, x) = L(y, x+1)
    dst[2][1:, :] = src[3][:-1, :]     # U'(y, x) = D(y-1, x)
    dst[3][:-1, :] = src[2][1:, :]     # D'(y, x) = U(y+1, x)
    return admit(GridGraph(W, H, g.snk_cap.copy(), g.src_cap.copy(), dst.reshape(4, -1)))


def _plan(widths, heights, pad):
    """Segment offsets / bridge columns / height of a left-to-right join."""
    height = max(heights)
    if not pad and any(h != height for h in heights):
        raise SupergraphError(f"height mismatch {sorted(set(heights))}; pass pad=True to pad")
    offsets, bridges, col = [], [], 0
    for i, w in enumerate(widths):
        offsets.append(col)
        col += w
        if i + 1 < len(widths):
            bridges.append(col)
            col += 1
    return offsets, bridges, height, col


def join(graphs, swapped=None, pad=False):
    """Knit graphs left to right, one zero-capacity bridge column between
    neighbours; shorter graphs are zero-padded at the bottom when ``pad``.
    ``swapped`` only records how the caller embedded each constituent."""
    graphs = list(graphs)
    if not graphs:
        raise SupergraphError("join needs at least one graph")
    flags = [False] * len(graphs) if swapped is None else [bool(s) for s in swapped]
    if len(flags) != len(graphs):
        raise SupergraphError("swapped flags must match the graph count")
    offsets, bridges, height, total_w = _plan([g.width for g in graphs],
                                              [g.height for g in graphs], pad)
    planes = np.zeros((6, height, total_w), np.int64)   # src, snk, L, R, U, D
    for g, off in zip(graphs, offsets):
        block = np.concatenate([g.src_cap[None], g.snk_cap[None], g.nbr_cap])
        planes[:, :g.height, off:off + g.width] = block.reshape(6, g.height, g.width)
    flat = planes.reshape(6, -1)
    composite = admit(GridGraph(total_w, height, flat[0], flat[1], flat[2:]))
    segs = tuple(Segment(i, o, g.width, f) for i, (g, o, f) in enumerate(zip(graphs, offsets, flags)))
    return composite, SupergraphLayout(segs, tuple(bridges), height)


def split(layout: SupergraphLayout, composite: CutResult, graphs) -> list:
    """Per-constituent cuts from a composite cut; swapped spans are
    complemented, padding rows dropped, flows recomputed by cut_cost and
    checked to add up to the composite flow."""
    graphs = list(graphs)
    if len(graphs) != len(layout.segments):
        raise SupergraphError("graph count does not match the layout")
    n = layout.total_width * layout.height
    if composite.labels.size != n:
        raise SupergraphError(
            f"composite labels have {composite.labels.size} entries, layout implies {n}")
    grid = composite.labels.reshape(layout.height, layout.total_width)
    parts = []
    for seg, g in zip(layout.segments, graphs):
        if g.width != seg.width or g.height > layout.height:
            raise SupergraphError(f"constituent {seg.constituent} does not fit its segment")
        span = grid[:g.height, seg.offset:seg.offset + seg.width]
        lab = np.ascontiguousarray((1 - span) if seg.swapped else span, dtype=np.uint8).reshape(-1)
        parts.append(CutResult(cut_cost(g, lab), lab))
    total = sum(p.flow for p in parts)
    if total != composite.flow:
        raise SupergraphError(
            f"decoded flows sum to {total}, composite flow is {composite.flow}; "
            "the composite labels are not an optimal cut")
    return parts


def _segments_of(layout):
    if layout is None:
        return None
    return [(s.offset, s.width, s.swapped) for s in layout.segments]


def solve_composite(g: GridGraph, layout: SupergraphLayout | None = None,
                    device: int = 0) -> CutResult:
    """Solve a (possibly composite) graph on the GPU.

    Unswapped spans report the minimal source side; swapped spans report the
    complement of the sink-reaching set (supergraph.py:201-206), so ``split``
    lands every constituent on its original canonical cut."""
    from . import _native
    admit(g)
    (flow, labels), = _native.solver_for_thread(device).solve_composites(
        [(g.width, g.height, g.src_cap, g.snk_cap, g.nbr_cap, _segments_of(layout))])
    return CutResult(flow, labels)


def solve_composites(tasks, device: int = 0) -> list:
    """Batch form of solve_composite: [(graph, layout)] -> [CutResult], all
    in one device solve."""
    from . import _native
    items = []
    for g, layout in tasks:
        admit(g)
        items.append((g.width, g.height, g.src_cap, g.snk_cap, g.nbr_cap, _segments_of(layout)))
    return [CutResult(f, l) for f, l in _native.solver_for_thread(device).solve_composites(items)]


def family_swap_decision(problem: SeedProblem, schedule: LambdaSchedule) -> bool:
    """One swap decision per lambda family, taken at mid-schedule."""
    return swap_decision(instantiate(problem, schedule[schedule.mid_index]))


def build_lambda_supergraph(problem: SeedProblem, schedule: LambdaSchedule, swap: bool):
    """(composite, layout, originals) of one problem's lambda family."""
    originals = [instantiate(problem, lam) for lam in schedule]
    embedded = [apply_swap(g) for g in originals] if swap else originals
    composite, layout = join(embedded, swapped=[swap] * len(originals))
    return composite, layout, originals


def _check_seed_args(problems, swap_mode):
    problems = list(problems)
    if not problems:
        raise SupergraphError("need at least one problem")
    if swap_mode not in ("auto", "on", "off"):
        raise SupergraphError(f"unknown swap_mode {swap_mode!r}")
    return problems


def build_seed_supergraph(problems, schedule: LambdaSchedule, swap_mode: str = "auto"):
    """Host composite of several problems' lambda families (problem-major,
    lambda-minor), each with its own swap decision."""
    problems = _check_seed_args(problems, swap_mode)
    originals, embedded, flags = [], [], []
    for p in problems:
        swap = family_swap_decision(p, schedule) if swap_mode == "auto" else swap_mode == "on"
        for lam in schedule:
            g = instantiate(p, lam)
            originals.append(g)
            embedded.append(apply_swap(g) if swap else g)
            flags.append(swap)
    composite, layout = join(embedded, swapped=flags)
    return composite, layout, originals


_SKELETONS = {}
_SKEL_LOCK = threading.Lock()


def _layout_skeleton(problems, schedule: LambdaSchedule):
    """Segments -- unswapped and swapped instances of every one -- bridge
    columns and height of the layout build_seed_supergraph would produce.
    Segment is immutable, so the instances are cached per batch shape and
    shared by every layout of that shape (a C5 batch has 16,000 segments)."""
    k = len(schedule)
    shapes = [(p.width, p.height) for p in problems]
    key = (shapes[0], len(shapes), k) if len(set(shapes)) == 1 else (tuple(shapes), k)
    with _SKEL_LOCK:
        hit = _SKELETONS.get(key)
    if hit is not None:
        return hit
    widths = [w for (w, _) in shapes for _ in range(k)]
    offsets, bridges, height, _ = _plan(widths, [h for (_, h) in shapes for _ in range(k)], False)
    new = object.__new__
    variants = []
    for sw in (False, True):
        segs = []
        for i, (o, w) in enumerate(zip(offsets, widths)):
            seg = new(Segment)                     # frozen dataclass, fields set directly
            seg.__dict__.update(constituent=i, offset=o, width=w, swapped=sw)
            segs.append(seg)
        variants.append(tuple(segs))
    sk = (variants[0], variants[1], tuple(bridges), height)
    with _SKEL_LOCK:
        if len(_SKELETONS) >= 16:
            _SKELETONS.pop(next(iter(_SKELETONS)))
        _SKELETONS[key] = sk
    return sk


def _finish_layout(skeleton, swapped, k: int) -> SupergraphLayout:
    plain, swapped_segs, bridges, height = skeleton
    flags = np.asarray(swapped, bool)
    if not flags.any():
        return SupergraphLayout(plain, bridges, height)
    segs = list(plain)
    for i in np.flatnonzero(flags):   # a swapped family: its k segments
        segs[i * k:(i + 1) * k] = swapped_segs[i * k:(i + 1) * k]
    return SupergraphLayout(tuple(segs), bridges, height)


def seed_layout(problems, schedule: LambdaSchedule, swapped) -> SupergraphLayout:
    """The layout build_seed_supergraph would produce for these problems."""
    return _finish_layout(_layout_skeleton(problems, schedule), swapped, len(schedule))


@dataclass(frozen=True, eq=False)
class SeedSupergraphResult:
    """Device result of one seed supergraph: its layout and the decoded
    per-constituent cuts (problem-major, lambda-minor)."""

    layout: SupergraphLayout
    cuts: tuple
    scores: tuple = ()   # scoring.CutScore per cut when truths were given

    @property
    def flow(self) -> int:
        return sum(c.flow for c in self.cuts)


def check_seed_supergraph(problems, schedule: LambdaSchedule, swap_mode: str = "auto"):
    """Raise whatever build_seed_supergraph would raise, in the same order."""
    problems = _check_seed_args(problems, swap_mode)
    shapes = {(p.width, p.height) for p in problems}
    prefetch_family_stats(problems)
    for p in problems:
        if swap_mode == "auto":
            check_family(p, (schedule[schedule.mid_index],))
        check_family(p, schedule.values)
    if len({h for _, h in shapes}) > 1:
        raise SupergraphError(f"height mismatch {sorted({h for _, h in shapes})}; "
                              "pass pad=True to pad")
    return problems


def _stage_checked(solver, problems, schedule: LambdaSchedule, swap_mode: str) -> None:
    """Stage one same-shape seed batch on ``solver``: the admission checks
    (Python, the reference's errors in order) run while the engine narrows
    and copies the planes on a host thread (its ctypes call releases the
    GIL); a check error wins over a staging error."""
    W, H = problems[0].width, problems[0].height
    staged = {}

    def stage():
        try:
            solver.seed_stage(W, H, problems, schedule.values, swap_mode)
        except BaseException as exc:  # noqa: BLE001 -- re-raised below
            staged["err"] = exc

    sth = threading.Thread(target=stage)
    sth.start()
    try:
        check_seed_supergraph(problems, schedule, swap_mode)
    finally:
        sth.join()
    if "err" in staged:
        raise staged["err"]


def _collect(solver, problems, schedule: LambdaSchedule, skeleton, truths) -> SeedSupergraphResult:
    """Results of the batch the solver last ran: D2H of flows and label bits
    (unpacked on the host cores), device scores, CutResults and layout."""
    swapped, flows, labels = solver.seed_fetch(True)
    scores = ()
    if truths is not None:
        from .scoring import score_cuts
        scores = score_cuts(solver, truths)
    return _result(problems, schedule, skeleton, swapped, flows, labels, scores)


def _result(problems, schedule, skeleton, swapped, flows, labels, scores) -> SeedSupergraphResult:
    fl = np.asarray(flows).tolist() if isinstance(flows, np.ndarray) else [[int(f) for f in r] for r in flows]
    cuts = tuple(CutResult._trusted(fl[i][j], labels[i][j])
                 for i in range(len(problems)) for j in range(len(schedule)))
    layout = (_finish_layout(skeleton, swapped, len(schedule)) if skeleton is not None
              else seed_layout(problems, schedule, swapped))
    return SeedSupergraphResult(layout, cuts, scores)


def _solve_mixed(solver, problems, schedule: LambdaSchedule, swap_mode: str, truths, after=None):
    """Problems of one height and several widths: one device batch per
    width (the first run waits for ``after``'s last launched run)."""
    check_seed_supergraph(problems, schedule, swap_mode)
    if truths is not None:
        raise SupergraphError("device scoring needs problems of one shape")
    shapes = {(p.width, p.height) for p in problems}
    swapped = np.zeros(len(problems), bool)
    flows = [None] * len(problems)
    labels = [None] * len(problems)
    for (W, H) in sorted(shapes):
        idx = [i for i, p in enumerate(problems) if (p.width, p.height) == (W, H)]
        solver.seed_stage(W, H, [problems[i] for i in idx], schedule.values, swap_mode)
        solver.seed_launch(after)
        solver.seed_wait()
        after = None
        sw, fl, lb = solver.seed_fetch(True)
        for k, i in enumerate(idx):
            swapped[i], flows[i], labels[i] = sw[k], fl[k], lb[k]
    return _result(problems, schedule, None, swapped, flows, labels, ())


def solve_seed_supergraph(problems, schedule: LambdaSchedule, swap_mode: str = "auto",
                          device: int = 0, truths=None) -> SeedSupergraphResult:
    """Build + solve + decode a seed supergraph entirely on the device.
    With ``truths`` (one 0/1 mask per problem) every cut is also scored on
    the device (foreground count, exact overlap; harness/bench.py:95-113)."""
    from . import _native
    problems = _check_seed_args(problems, swap_mode)
    solver = _native.solver_for_thread(device)
    if len({(p.width, p.height) for p in problems}) != 1:
        with _native.device_lock(device):
            return _solve_mixed(solver, problems, schedule, swap_mode, truths)
    _stage_checked(solver, problems, schedule, swap_mode)
    # the layout's Segment objects (~3 us each in Python; 8,000 for a C5
    # batch) are built on a host thread while the device solves (the
    # engine's ctypes calls release the GIL); swap flags are set after
    box = {}
    th = None
    if len(problems) * len(schedule) >= 512:   # small layouts: not worth a thread
        th = threading.Thread(target=lambda: box.update(sk=_layout_skeleton(problems, schedule)))
        th.start()
    try:
        with _native.device_lock(device):
            solver.seed_run()
    finally:
        if th is not None:
            th.join()
    return _collect(solver, problems, schedule, box.get("sk"), truths)


def solve_seed_supergraphs(batches, schedule: LambdaSchedule, swap_mode: str = "auto",
                           device: int = 0, truths=None, depth: int = 3, overlap_us: int = 20):
    """Stream of seed supergraphs through one device: yields, in order, what
    ``solve_seed_supergraph(batch, schedule, swap_mode, device, truths_k)``
    returns for each batch (a list of problems, or a synth_device.ImageBatch
    whose planes the device derives) of ``batches`` -- same values, same
    errors.  ``truths`` is None or an iterable with one list of
    truth masks (or None) per batch.

    The host work of neighbouring batches overlaps the device: a stager
    thread admits and stages batch k + 1 (narrowing, H2D) on the next of
    ``depth`` solvers of the device while batch k runs, and launches it at
    once behind the previous run (pmf_seed_launch with `after`: runs never
    share the GPU and start back to back with no host round trip in
    between); the caller's thread waits for batch k, fetches and decodes it
    (D2H, label unpack, CutResults) while batch k + 1 runs.  An error of
    batch k is raised when its result is due; the stream ends there.  The
    serving analogue of run_dynamic's per-worker slots
    (scheduler.py:253-292, harness/bench.py:79-93).

    ``overlap_us`` (0: off): two consecutive batches that both run on the
    asynchronous solver (small batches, C1-C3) may share the device -- the
    later run starts once the one before the previous has finished, and the
    idle CTAs of a run's latency-bound tail leave the SM to it after that
    many microseconds of an empty queue (knob async_yield_us).  Step-
    synchronous runs (cooperative launches) never share the device.  A stream owns its
    solvers (nested streams of one thread lease separate ones) and expects
    no concurrent solves on its device from other threads."""
    import queue

    from . import _native
    from .synth_device import ImageBatch, stage_image_batch
    if depth < 2:
        raise ValueError("depth must be >= 2")
    solvers = _native.pipeline_solvers(device, depth + 1, lease=True)
    mixed = solvers[depth]   # mixed-width batches, solved synchronously by the stager
    for sv in solvers:
        sv.set("async_yield_us", overlap_us)

    def launch(sv, prev):
        """Launch sv's staged run behind every other solver's last run --
        except the previous one when both runs are asynchronous (they may
        share the device)."""
        share = (overlap_us > 0 and prev is not None and prev is not sv and sv.seed_kind()[0]
                 and prev.seed_kind()[1])
        for o in solvers:
            if o is not sv and not (share and o is prev):
                sv.depend(o)
        sv.seed_launch(None)
    free = [threading.Semaphore(1) for _ in range(depth)]
    to_fetch = queue.Queue()
    stop = threading.Event()

    def stager():
        prev = None   # solver of the last launched run
        try:
            tr_iter = iter(truths) if truths is not None else None
            for k, probs in enumerate(batches):
                tr = next(tr_iter) if tr_iter is not None else None
                slot = k % depth
                free[slot].acquire()   # the slot's previous batch has been fetched
                if stop.is_set():
                    return
                sv = solvers[slot]
                try:
                    if isinstance(probs, ImageBatch):   # planes derived on the device
                        fams = stage_image_batch(sv, probs, schedule, swap_mode)
                        item = ("ok", (fams, _layout_skeleton(fams, schedule)), tr)
                    else:
                        probs = _check_seed_args(probs, swap_mode)
                        if len({(p.width, p.height) for p in probs}) != 1:
                            item = ("done", _solve_mixed(mixed, probs, schedule, swap_mode, tr, prev), None)
                            prev = mixed
                        else:
                            _stage_checked(sv, probs, schedule, swap_mode)
                            item = ("ok", (probs, _layout_skeleton(probs, schedule)), tr)
                    if item[0] == "ok":
                        launch(sv, prev)
                        prev = sv
                except BaseException as exc:  # noqa: BLE001 -- raised by the consumer
                    item = ("err", exc, None)
                to_fetch.put((slot, item))
        except BaseException as exc:  # noqa: BLE001 -- batches / truths iterables raised
            to_fetch.put((None, ("err", exc, None)))
        to_fetch.put(None)

    th = threading.Thread(target=stager, daemon=True)
    th.start()
    try:
        while True:
            x = to_fetch.get()
            if x is None:
                return
            slot, (kind, a, tr) = x
            try:
                if kind == "err":
                    raise a
                if kind == "done":
                    res = a
                else:
                    s = solvers[slot]
                    s.seed_wait()
                    res = _collect(s, a[0], schedule, a[1], tr)
            finally:
                if slot is not None:
                    free[slot].release()
            yield res
            del res
    finally:
        stop.set()
        for f in free:
            f.release()
        th.join()
        for s in solvers:   # a run launched but never waited for (stream closed early)
            s.abandon()
        _native.release_solvers(device, solvers)
