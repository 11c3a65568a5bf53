"""Parametric seed problems and lambda schedules.

Mirror of /root/reference/pkg/src/pmflow/parametric.py: ``LambdaSchedule``
(:41-77), ``SeedProblem`` (:80-130), ``instantiate`` (:133-166),
``solve_schedule_sequential`` (:180-183), ``energy`` (:186-188),
``check_nested`` (:191-201), same errors.

Device path: ``solve_schedule_sequential`` builds every lambda graph on the
GPU from the problem planes and solves them as one batch (the "batch"
baseline of the paper without the per-call overhead).  ``check_family``
reproduces, without materialising any graph, every error ``instantiate``
would raise for a list of lambdas, in the reference's order, so the device
builder only ever sees admissible problems.
"""

from __future__ import annotations

import os
import threading
import weakref
from dataclasses import dataclass, field

import numpy as np

from .grid import (CAP_MAX, BorderEdgeError, CapacityOverflowError, CutResult, GridGraph,
                   NegativeCapacityError, ShapeError, TOTAL_CAP_LIMIT, admit, cut_cost)

DEFAULT_LAMBDA_VALUES = (1, 2, 3, 5, 7, 11, 16, 24, 36, 54,
                         81, 122, 183, 274, 411, 617, 925, 1388, 2082, 3123)
HALVED_LAMBDA_VALUES = DEFAULT_LAMBDA_VALUES[::2]

_PRODUCT_LIMIT = 1 << 62


class ScheduleError(ValueError):
    pass


class ProblemError(ValueError):
    pass


@dataclass(frozen=True)
class LambdaSchedule:
    """Strictly increasing non-negative integer lambda values."""

    values: tuple

    def __post_init__(self):
        vals = tuple(int(v) for v in self.values)
        if not vals:
            raise ScheduleError("schedule must hold at least one value")
        if vals[0] < 0:
            raise ScheduleError("lambda values must be non-negative")
        if any(b <= a for a, b in zip(vals, vals[1:])):
            raise ScheduleError("lambda values must be strictly increasing")
        object.__setattr__(self, "values", vals)

    @classmethod
    def default(cls) -> "LambdaSchedule":
        return cls(DEFAULT_LAMBDA_VALUES)

    @classmethod
    def halved(cls) -> "LambdaSchedule":
        return cls(HALVED_LAMBDA_VALUES)

    @property
    def mid_index(self) -> int:
        """ceil(n/2) - 1: the value the family swap decision is taken at."""
        return (len(self.values) - 1) // 2

    def __len__(self):
        return len(self.values)

    def __iter__(self):
        return iter(self.values)

    def __getitem__(self, i):
        return self.values[i]


@dataclass(frozen=True, eq=False)
class SeedProblem:
    """Unary/pairwise terms plus foreground/background seed pixels."""

    width: int
    height: int
    unary_base: np.ndarray
    unary_slope: np.ndarray
    sink_base: np.ndarray
    pairwise: np.ndarray  # (4, n), LEFT/RIGHT/UP/DOWN rows
    fg_seeds: frozenset = field(default_factory=frozenset)
    bg_seeds: frozenset = field(default_factory=frozenset)

    def __post_init__(self):
        if self.width < 1 or self.height < 1:
            raise ProblemError(f"bad dimensions {self.width}x{self.height}")
        n = self.width * self.height
        set_ = object.__setattr__
        for name in ("unary_base", "unary_slope", "sink_base"):
            a = np.asarray(getattr(self, name), dtype=np.int64).reshape(-1)
            if a.size != n:
                raise ShapeError(f"{name}: expected {n} entries, got {a.size}")
            set_(self, name, a)
        pw = np.asarray(self.pairwise, dtype=np.int64)
        if pw.size != 4 * n:
            raise ShapeError(f"pairwise: expected shape (4, {n}), got {pw.shape}")
        set_(self, "pairwise", pw.reshape(4, n))
        if self.unary_slope.size and int(self.unary_slope.min()) < 0:
            raise ProblemError("unary_slope must be non-negative")
        fg, fg_idx = _seed_set(self.fg_seeds)
        bg, bg_idx = _seed_set(self.bg_seeds)
        if fg & bg:
            raise ProblemError("a pixel cannot be both a foreground and background seed")
        for name, idx in (("fg_seeds", fg_idx), ("bg_seeds", bg_idx)):
            if idx.size and (int(idx[0]) < 0 or int(idx[-1]) >= n):
                raise ProblemError(f"{name} contains an out-of-range pixel index")
        set_(self, "fg_seeds", fg)
        set_(self, "bg_seeds", bg)
        set_(self, "_fg_idx", fg_idx)
        set_(self, "_bg_idx", bg_idx)
        set_(self, "_stats", None)

    @property
    def n(self) -> int:
        return self.width * self.height

    def _family_stats(self):
        """Lambda-independent reductions used by check_family (cached).

        Whole-plane reductions come from a cache keyed by the plane's memory
        (``_plane_stats``): the problems of one image share its pairwise
        plane and the seed types of one seed share their unary / sink planes,
        so a CPMC image's 50 problems reduce 26 distinct planes, not 200.
        The seed pixels are then taken out exactly (sums) or bounded (the
        extrema only gate exact fallbacks, _check_lambda)."""
        if self._stats is None:
            fg, bg = self._fg_idx, self._bg_idx
            b, s, sink, pw = self.unary_base, self.unary_slope, self.sink_base, self.pairwise
            sb, ss, sk = _plane_stats(b), _plane_stats(s), _plane_stats(sink)
            sp = _plane_stats(pw, self.height, self.width)
            kb = sink[bg]
            st = dict(
                max_slope=ss["max"], max_base=sb["max"],
                # bounds over all pixels (>= the non-seed extrema): a bound that
                # passes implies the exact value passes; otherwise exact below
                min_base_nonfg=sb["min"] if sb["min"] >= 0 else
                int(b[self._nonfg()].min(initial=0)),
                sum_base_nonfg=sb["sum"] - int(b[fg].sum()),
                sum_slope_nonfg=ss["sum"] - int(s[fg].sum()),
                max_slope_nonfg=ss["max"], max_base_nonfg=sb["max"],
                n_fg=int(fg.size), n_bg=int(bg.size),
                min_sink=sk["min"] if sk["min"] >= 0 else int(sink[self._nonbg()].min(initial=0)),
                max_sink=sk["max"] if sk["max"] <= CAP_MAX else int(sink[self._nonbg()].max(initial=0)),
                sum_sink=sk["sum"] - int(kb.sum()),
                sum_sink_fin=sk["sum_fin"] - int(kb[kb < CAP_MAX].sum()),
                min_pw=sp["min"], max_pw=sp["max"], sum_pw=sp["sum"], sum_pw_fin=sp["sum_fin"],
                border=sp["border"],
            )
            object.__setattr__(self, "_stats", st)
        return self._stats

    def _nonfg(self):
        m = np.ones(self.n, bool)
        m[self._fg_idx] = False
        return m

    def _nonbg(self):
        m = np.ones(self.n, bool)
        m[self._bg_idx] = False
        return m


_SEED_SETS = {}
_PRUNE_AT = {}


def _prune(cache: dict) -> None:
    """Drop the entries whose object died, once the cache has doubled since
    the last pass (amortised O(1) per insertion even when every cached
    object is still alive, e.g. many batches of problems held at once)."""
    limit = _PRUNE_AT.get(id(cache), 4096)
    if len(cache) <= limit:
        return
    for k in [k for k, (r, _) in cache.items() if r() is None]:
        del cache[k]
    _PRUNE_AT[id(cache)] = max(4096, 2 * len(cache))


def _seed_set(seeds):
    """(frozenset of int, sorted read-only int64 index array) of a seed set.
    A frozenset of Python ints seen before (the problems of one image share
    their border background set) is reused as is, with its index array."""
    if isinstance(seeds, frozenset):
        ent = _SEED_SETS.get(id(seeds))
        if ent is not None and ent[0]() is seeds:
            return seeds, ent[1]
    fs = frozenset(int(i) for i in seeds)
    idx = np.fromiter(sorted(fs), np.int64, len(fs))
    idx.flags.writeable = False
    if isinstance(seeds, frozenset) and len(fs) > 64 and all(type(i) is int for i in seeds):
        with _PLANE_LOCK:
            _prune(_SEED_SETS)
            _SEED_SETS[id(seeds)] = (weakref.ref(seeds), idx)
        return seeds, idx
    return fs, idx


_PLANE_STATS = {}
_PLANE_LOCK = threading.Lock()


def _plane_stats(a: np.ndarray, height: int = 0, width: int = 0, pre: dict | None = None) -> dict:
    """min / max / sum / sum below CAP_MAX of a plane (and, for a (4, n)
    pairwise plane with height/width, the largest arc on each image border),
    cached by the plane's memory while an array viewing it is alive."""
    key = (a.__array_interface__["data"][0], a.shape, a.dtype.str, height, width)
    with _PLANE_LOCK:
        ent = _PLANE_STATS.get(key)
        if ent is not None and ent[0]() is not None:
            return ent[1]
    if pre is not None:
        st = dict(pre)
    else:
        st = dict(min=int(a.min(initial=0)), max=int(a.max(initial=0)), sum=int(a.sum()))
        st["sum_fin"] = st["sum"] if st["max"] < CAP_MAX else int(a[a < CAP_MAX].sum())
    if height:
        arcs = a.reshape(4, height, width)
        st["border"] = [(d, int(row.max(initial=0))) for d, row in (
            (0, arcs[0][:, 0]), (1, arcs[1][:, -1]), (2, arcs[2][0, :]), (3, arcs[3][-1, :]))]
    with _PLANE_LOCK:
        _prune(_PLANE_STATS)
        _PLANE_STATS[key] = (weakref.ref(a), st)
    return st


def prefetch_family_stats(problems) -> None:
    """Reduce the distinct planes of many problems on a thread pool (numpy
    releases the GIL in its reductions): a batch of CPMC images has hundreds
    of planes, which one thread reduces at ~1 GB/s."""
    todo, seen = [], set()
    for p in problems:
        if getattr(p, "_stats", None) is not None:
            continue
        for a, hw in ((p.unary_base, None), (p.unary_slope, None), (p.sink_base, None),
                      (p.pairwise, (p.height, p.width))):
            key = (a.__array_interface__["data"][0], a.shape)
            if key not in seen:
                seen.add(key)
                todo.append((a, hw))
    if len(todo) < 8 and sum(a.size for a, _ in todo) < (1 << 20):
        return   # a few small planes: numpy is quicker than a native pool round trip
    try:
        from ._native import plane_stats
        red = plane_stats([a for a, _ in todo])
    except Exception:  # noqa: BLE001 -- library not built: numpy per plane below
        return
    for (a, hw), (mn, mx, sm, fin) in zip(todo, red):
        _plane_stats(a, *(hw or ()), pre=dict(min=mn, max=mx, sum=sm, sum_fin=fin))


def _check_lambda(p: SeedProblem, lam: int) -> None:
    """Raise exactly what instantiate(p, lam) raises (parametric.py:141-165
    and admit, grid.py:112-126), or return if the graph is admissible."""
    lam = int(lam)
    if lam < 0:
        raise ScheduleError(f"lambda must be non-negative, got {lam}")
    st = p._family_stats()
    if st["max_slope"] and lam > _PRODUCT_LIMIT // st["max_slope"]:
        raise CapacityOverflowError(f"lambda {lam} overflows the unary term")
    exact = st["max_base"] + lam * st["max_slope"] > CAP_MAX
    src_all = None
    if exact:
        src_all = p.unary_base + lam * p.unary_slope
        over = src_all > CAP_MAX
        if bool(over.any()):
            raise CapacityOverflowError(
                f"unary_base + lambda*unary_slope exceeds CAP_MAX at pixel {int(np.argmax(over))} "
                f"(lambda={lam})")
    # admit on the instantiated graph: src (fg pixels are CAP_MAX)
    if st["min_base_nonfg"] < 0:
        nonfg = p._nonfg()
        src_nf = p.unary_base[nonfg] + lam * p.unary_slope[nonfg]
        if src_nf.size and int(src_nf.min()) < 0:
            raise NegativeCapacityError("src_cap has a negative capacity")
    if st["min_sink"] < 0:
        raise NegativeCapacityError("snk_cap has a negative capacity")
    if st["max_sink"] > CAP_MAX:
        raise CapacityOverflowError("snk_cap exceeds CAP_MAX = 2**30")
    if st["min_pw"] < 0:
        raise NegativeCapacityError("nbr_cap has a negative capacity")
    if st["max_pw"] > CAP_MAX:
        raise CapacityOverflowError("nbr_cap exceeds CAP_MAX = 2**30")
    for d, m in st["border"]:
        if m > 0:
            raise BorderEdgeError(f"nonzero {('left', 'right', 'up', 'down')[d]} capacity on the "
                                  "image border")
    src_sum = st["sum_base_nonfg"] + lam * st["sum_slope_nonfg"] + st["n_fg"] * CAP_MAX
    total = src_sum + st["sum_sink"] + st["n_bg"] * CAP_MAX + st["sum_pw"]
    if total >= TOTAL_CAP_LIMIT:
        raise CapacityOverflowError("total capacity exceeds the 2**62 admission budget")
    # seed headroom (parametric.py:160-165)
    if st["max_base_nonfg"] + lam * st["max_slope_nonfg"] < CAP_MAX:
        src_fin = st["sum_base_nonfg"] + lam * st["sum_slope_nonfg"]
    else:
        nonfg = p._nonfg()
        s_nf = p.unary_base[nonfg] + lam * p.unary_slope[nonfg]
        src_fin = int(s_nf[s_nf < CAP_MAX].sum())
    finite = src_fin + st["sum_sink_fin"] + st["sum_pw_fin"]
    if finite >= CAP_MAX:
        raise CapacityOverflowError(
            f"finite capacities sum to {finite}, leaving no headroom under CAP_MAX; "
            "seed pixels could be severed")


def check_family(problem: SeedProblem, lambdas) -> None:
    """Raise the first error instantiate() would raise over ``lambdas`` (in
    order); the device builder relies on this having passed.

    Fast path: when no non-seed unary term is negative and no source
    capacity reaches CAP_MAX at the largest lambda, every check of
    _check_lambda is monotone in lambda (capacities only grow with lambda
    and the finite-capacity sum is linear in it), so an increasing schedule
    passes iff its largest value passes.  Otherwise (or if it fails) the
    values are checked in order, which finds the reference's first error."""
    lambdas = list(lambdas)
    if not lambdas:
        return
    lam_max = max(int(v) for v in lambdas)
    st = problem._family_stats()
    if (lam_max >= 0 and st["min_base_nonfg"] >= 0 and
            (not st["max_slope"] or lam_max <= _PRODUCT_LIMIT // st["max_slope"]) and
            st["max_base"] + lam_max * st["max_slope"] < CAP_MAX and
            all(int(v) >= 0 for v in lambdas)):
        try:
            _check_lambda(problem, lam_max)
            return
        except (CapacityOverflowError, NegativeCapacityError, BorderEdgeError, ScheduleError):
            pass
    for lam in lambdas:
        _check_lambda(problem, lam)


def instantiate(problem: SeedProblem, lam: int) -> GridGraph:
    """Host-built admitted graph for one lambda value (API compatibility;
    the device path never materialises it)."""
    _check_lambda(problem, lam)
    src = problem.unary_base + int(lam) * problem.unary_slope
    snk = problem.sink_base.copy()
    src[problem._fg_idx] = CAP_MAX
    snk[problem._bg_idx] = CAP_MAX
    return admit(GridGraph(problem.width, problem.height, src, snk, problem.pairwise.copy()))


@dataclass(frozen=True, eq=False)
class ParametricResult:
    """Cuts for one problem at every schedule value, in order."""

    schedule: LambdaSchedule
    cuts: tuple

    def masks(self):
        return [c.labels.astype(bool) for c in self.cuts]


def solve_schedule_sequential(problem: SeedProblem, schedule: LambdaSchedule,
                              device: int = 0) -> ParametricResult:
    """Every lambda of the schedule solved independently (reference
    parametric.py:180-183), as one device batch of lambda graphs."""
    from . import _native
    check_family(problem, schedule.values)
    _, flows, labels = _native.solver_for_thread(device).solve_seed_batch(
        problem.width, problem.height, [problem], schedule.values, "off")
    return ParametricResult(schedule, tuple(CutResult(int(f), l)
                                            for f, l in zip(flows[0], labels[0])))


def energy(problem: SeedProblem, lam: int, labels) -> int:
    """Segmentation energy of a mask at one lambda (its cut cost)."""
    return cut_cost(instantiate(problem, lam), labels)


def check_nested(result: ParametricResult):
    """(True, None) if every mask contains its predecessor, else (False, i)
    for the first schedule index whose mask loses a pixel."""
    masks = result.masks()
    for i in range(1, len(masks)):
        if bool((masks[i - 1] & ~masks[i]).any()):
            return False, i
    return True, None
