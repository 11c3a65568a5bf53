"""On-device synthesis of CPMC seed batches.

The reference generates every seed problem's planes on the host
(/root/reference/pkg/src/pmflow/harness/synth.py:67-136, ``generate_batch``:
three unary/sink planes per seed and a pairwise plane per image, int64) and
ships them to the solver.  Here only the 8-bit images, the seed pixels and
the seed index lists cross the host link: the GPU derives the planes at the
start of the run (``pmf_synth_stage``; kernels ``k_synth_planes`` /
``k_synth_pw``), with the reference's integer arithmetic, so every cut is the
one ``solve_seed_supergraph`` returns for the host-built problems -- bit for
bit (tests/test_gpu_synth.py).

Admission (``instantiate``'s errors, parametric.py:133-166, in
``check_seed_supergraph`` order) runs on intensity histograms: a synthetic
problem's plane reductions are sums over 256 intensity bins, so
``ImageFamily`` hands ``check_family`` the exact statistics a materialised
``SeedProblem`` would (tests/test_synth_device.py pins them), and builds the
planes themselves only for the exact-value fallbacks near CAP_MAX.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, field

import numpy as np

from . import synth
from .parametric import LambdaSchedule, SeedProblem
from .supergraph import (SeedSupergraphResult, SupergraphError, _collect, _layout_skeleton,
                         check_seed_supergraph)

_DS = np.arange(256, dtype=np.int64)
_PW_LUT = 1 + ((synth.INTENSITY_MAX - _DS) * 63) // synth.INTENSITY_MAX   # arc value per |dI|
TYPES = ("A", "B")


class ImageFamily:
    """Stand-in for the SeedProblem of one (image, seed, type): the
    attributes check_family / _layout_skeleton read, statistics from
    histograms, planes built lazily (only the exact fallbacks need them)."""

    def __init__(self, img, x, y, bg, bg_idx, stats):
        self.height, self.width = img.shape
        self._img, self._x, self._y = img, x, y
        self.fg_seeds = frozenset({y * self.width + x})
        self.bg_seeds = bg
        self._fg_idx = np.array([y * self.width + x], np.int64)
        self._bg_idx = bg_idx
        self._stats = stats
        self._planes = None

    @property
    def n(self) -> int:
        return self.width * self.height

    def _family_stats(self):
        return self._stats

    def _terms(self):
        if self._planes is None:
            self._planes = synth.seed_terms(self._img, self._x, self._y)
        return self._planes

    @property
    def unary_base(self):
        return self._terms()[0]

    @property
    def unary_slope(self):
        return self._terms()[1]

    @property
    def sink_base(self):
        return self._terms()[2]

    @property
    def pairwise(self):
        return synth.contrast_weights(self._img)

    def _nonfg(self):
        m = np.ones(self.n, bool)
        m[self._fg_idx] = False
        return m

    def _nonbg(self):
        m = np.ones(self.n, bool)
        m[self._bg_idx] = False
        return m

    def problem(self) -> SeedProblem:
        """The host SeedProblem this family stands for (synth.seed_problem)."""
        return SeedProblem(width=self.width, height=self.height, unary_base=self.unary_base,
                           unary_slope=self.unary_slope, sink_base=self.sink_base, pairwise=self.pairwise,
                           fg_seeds=self.fg_seeds, bg_seeds=self.bg_seeds)


def _ring(width, height, top=True):
    """Row-major indices of the border (without its top row if not top)."""
    return synth.border_pixels(width, height, top)


def image_family_stats(img, x, y, bg_idx, hist=None, edge_hist=None) -> dict:
    """check_family statistics of problem_for_seed(img, x, y) with background
    bg_idx, from intensity histograms (same values as
    SeedProblem._family_stats on the materialised planes)."""
    v = img.reshape(-1)
    if hist is None:
        hist = np.bincount(v, minlength=256)
    if edge_hist is None:
        edge_hist = (np.bincount(np.abs(np.diff(img, axis=1)).reshape(-1), minlength=256) +
                     np.bincount(np.abs(np.diff(img, axis=0)).reshape(-1), minlength=256))
    s = int(img[y, x])
    d = np.abs(_DS - s)
    base, slope, sink = (synth._TERM_LUT[k][d] for k in range(3))
    present = hist > 0
    bgh = np.bincount(v[bg_idx], minlength=256) if len(bg_idx) else np.zeros(256, np.int64)
    sum_b, sum_s, sum_k = (int(hist @ t) for t in (base, slope, sink))
    sink_bg = int(bgh @ sink)
    pw_present = edge_hist > 0
    max_pw = int(_PW_LUT[pw_present].max()) if pw_present.any() else 0
    sum_pw = 2 * int(edge_hist @ _PW_LUT)
    b0, s0 = int(synth._TERM_LUT[0][0]), int(synth._TERM_LUT[1][0])   # the fg seed: dsim 0
    return dict(
        max_slope=int(slope[present].max()), max_base=int(base[present].max()),
        min_base_nonfg=min(0, int(base[present].min())),   # reductions with initial=0, as _plane_stats
        sum_base_nonfg=sum_b - b0, sum_slope_nonfg=sum_s - s0,
        max_slope_nonfg=int(slope[present].max()), max_base_nonfg=int(base[present].max()),
        n_fg=1, n_bg=int(len(bg_idx)),
        min_sink=min(0, int(sink[present].min())), max_sink=int(sink[present].max()),
        sum_sink=sum_k - sink_bg, sum_sink_fin=sum_k - sink_bg,
        min_pw=0, max_pw=max_pw, sum_pw=sum_pw, sum_pw_fin=sum_pw,
        border=[(0, 0), (1, 0), (2, 0), (3, 0)],
    )


@dataclass
class ImageBatch:
    """Synthetic CPMC images whose seed problems are built on the device:
    ``images`` (k, H, W) intensities 0..255, the seed lattice ``coords``
    [(x, y)] shared by every image, seed ``types`` ("A": border background,
    "B": border minus the top row), optional region maps for truths.
    Problems are image-major, seed, type-minor (synth.generate's order,
    image after image)."""

    images: np.ndarray
    coords: list
    types: tuple = ("A",)
    regions: np.ndarray | None = None
    _fams: list | None = field(default=None, repr=False)

    def __post_init__(self):
        imgs = np.asarray(self.images)
        if imgs.ndim != 3:
            raise ValueError("images must be (count, height, width)")
        if imgs.size and (int(imgs.min()) < 0 or int(imgs.max()) > synth.INTENSITY_MAX):
            raise ValueError("intensities must lie in [0, 255]")
        self.images = imgs
        self.types = tuple(self.types)
        if not self.types or any(t not in TYPES for t in self.types):
            raise ValueError(f"seed types must be among {TYPES}")

    @property
    def nimg(self) -> int:
        return int(self.images.shape[0])

    @property
    def height(self) -> int:
        return int(self.images.shape[1])

    @property
    def width(self) -> int:
        return int(self.images.shape[2])

    def families(self) -> list:
        """One ImageFamily per problem (admission and layout)."""
        if self._fams is None:
            W, H = self.width, self.height
            bgs = {"A": _ring(W, H), "B": _ring(W, H, top=False)}
            bidx = {t: np.fromiter(sorted(b), np.int64, len(b)) for t, b in bgs.items()}
            fams = []
            for img in self.images:
                img = np.asarray(img, np.int64)
                hist = np.bincount(img.reshape(-1), minlength=256)
                eh = (np.bincount(np.abs(np.diff(img, axis=1)).reshape(-1), minlength=256) +
                      np.bincount(np.abs(np.diff(img, axis=0)).reshape(-1), minlength=256))
                for (x, y) in self.coords:
                    for t in self.types:
                        if y * W + x in bgs[t]:
                            raise ValueError(f"seed ({x}, {y}) sits on the border")
                        st = image_family_stats(img, x, y, bidx[t], hist, eh)
                        fams.append(ImageFamily(img, x, y, bgs[t], bidx[t], st))
            self._fams = fams
        return self._fams

    def problems(self) -> list:
        """The host SeedProblems (what synth.generate builds for these images)."""
        return [f.problem() for f in self.families()]

    @property
    def truths(self) -> list:
        """Ground-truth mask per problem (its seed's region)."""
        if self.regions is None:
            raise ValueError("no region maps")
        return [synth.truth_mask(reg, x, y) for reg in self.regions for (x, y) in self.coords
                for _ in self.types]


def generate_images(width, height, seed_rows=1, seed_cols=1, rng_seeds=(0,), types=("A",), regions=4,
                    noise=10) -> ImageBatch:
    """Images of synth.generate(width, height, ..., rng_seed=s) for every s
    (the reference's rng stream, synth_image :22-41), without their planes."""
    imgs, regs = [], []
    for s in rng_seeds:
        img, reg = synth.draw_image(width, height, np.random.default_rng(s), regions, noise)
        imgs.append(img.astype(np.uint8))
        regs.append(reg)
    return ImageBatch(np.stack(imgs), synth.lattice(width, height, seed_rows, seed_cols), tuple(types),
                      np.stack(regs))


def stage_image_batch(solver, batch: ImageBatch, schedule: LambdaSchedule, swap_mode: str) -> list:
    """Admission checks (check_seed_supergraph on the families, the
    reference's errors in order) overlapping the engine's staging of the
    images; returns the families (layout order)."""
    if swap_mode not in ("auto", "on", "off"):
        raise SupergraphError(f"unknown swap_mode {swap_mode!r}")
    fams = batch.families()
    if not fams:
        raise SupergraphError("need at least one problem")
    staged = {}

    def stage():
        try:
            solver.synth_stage(batch.images, batch.coords, batch.types, schedule.values, swap_mode)
        except BaseException as exc:  # noqa: BLE001 -- re-raised below
            staged["err"] = exc

    th = threading.Thread(target=stage)
    th.start()
    try:
        check_seed_supergraph(fams, schedule, swap_mode)
    finally:
        th.join()
    if "err" in staged:
        raise staged["err"]
    return fams


def solve_image_batch(batch: ImageBatch, schedule: LambdaSchedule, swap_mode: str = "auto", device: int = 0,
                      truths=None) -> SeedSupergraphResult:
    """Seed supergraph of a batch of synthetic images, planes built on the
    device: the same result as solve_seed_supergraph(batch.problems(), ...)."""
    from . import _native
    solver = _native.solver_for_thread(device)
    fams = stage_image_batch(solver, batch, schedule, swap_mode)
    with _native.device_lock(device):
        solver.seed_run()
    return _collect(solver, fams, schedule, _layout_skeleton(fams, schedule), truths)
