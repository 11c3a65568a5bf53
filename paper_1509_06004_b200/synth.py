"""Benchmark inputs: the reference's synthetic seed problems, bit for bit.

Re-derivation of /root/reference/pkg/src/pmflow/harness/synth.py so the GPU
box (which has no reference checkout) generates the same problems from the
same ``rng_seed``: one image of random constant rectangles plus clipped
noise (synth.py:22-41), contrast-gated pairwise weights (:52-64), and one
seed problem per interior lattice point with the border as background
(:44-49, :73-100).  ``tests/test_oracle.py`` and ``tests/test_host.py`` pin
the planes against digests of the reference generator's problems.

CPMC seed "type B" (BASELINE.json config 3): the same
foreground seed with the border minus its top row as background -- not in
the reference; a documented SeedProblem variant.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .parametric import SeedProblem

INTENSITY_MAX = 255
L20 = (2, 3, 4, 5, 7, 9, 12, 16, 22, 30, 40, 54, 73, 99, 134, 181, 244, 329, 444, 600)
C4_LAMBDAS = (1, 2, 3, 5, 7, 11, 16, 24)


def draw_image(width, height, rng, regions=4, noise=10):
    """(image, region map), both (height, width) int64; rng draws in the
    reference's order: background, then per rectangle w, h, x0, y0, value,
    then the noise field."""
    img = np.full((height, width), int(rng.integers(0, INTENSITY_MAX + 1)), np.int64)
    reg = np.zeros((height, width), np.int64)
    for rid in range(1, regions + 1):
        rw = int(rng.integers(max(1, width // 4), max(2, 3 * width // 4)))
        rh = int(rng.integers(max(1, height // 4), max(2, 3 * height // 4)))
        x0 = int(rng.integers(0, max(1, width - rw + 1)))
        y0 = int(rng.integers(0, max(1, height - rh + 1)))
        img[y0:y0 + rh, x0:x0 + rw] = int(rng.integers(0, INTENSITY_MAX + 1))
        reg[y0:y0 + rh, x0:x0 + rw] = rid
    if noise:
        img = np.clip(img + rng.integers(-noise, noise + 1, (height, width)), 0, INTENSITY_MAX)
    return img, reg


def contrast_weights(img):
    """(4, n) pairwise capacities: 1 + 63 * (255 - |dI|) // 255 per edge,
    the same value on both arcs of an edge."""
    h, w = img.shape
    out = np.zeros((4, h, w), np.int64)
    horiz = 1 + ((INTENSITY_MAX - np.abs(np.diff(img, axis=1))) * 63) // INTENSITY_MAX
    vert = 1 + ((INTENSITY_MAX - np.abs(np.diff(img, axis=0))) * 63) // INTENSITY_MAX
    out[1][:, :-1] = horiz
    out[0][:, 1:] = horiz
    out[3][:-1, :] = vert
    out[2][1:, :] = vert
    return out.reshape(4, -1)


def lattice(width, height, rows, cols):
    """Interior seed points, row-major: y_i = (i+1)H/(rows+1), x_j likewise."""
    return [((j + 1) * width // (cols + 1), (i + 1) * height // (rows + 1))
            for i in range(rows) for j in range(cols)]


def border_pixels(width, height, top=True):
    grid = np.arange(width * height).reshape(height, width)
    ring = np.ones((height, width), bool)
    ring[1:-1, 1:-1] = False
    if not top:
        ring[0, :] = False
    return frozenset(int(p) for p in grid[ring])


# the three terms of every intensity difference dsim = |I - I(seed)| in
# [0, 255]: base 1 + 15 (255 - dsim) // 255, slope 1 + 7 (255 - dsim) // 255,
# sink 1 + 63 dsim // 255 (harness/synth.py seed terms), as lookup tables
_DS = np.arange(INTENSITY_MAX + 1, dtype=np.int64)
_TERM_LUT = np.stack([1 + ((INTENSITY_MAX - _DS) * 15) // INTENSITY_MAX,
                      1 + ((INTENSITY_MAX - _DS) * 7) // INTENSITY_MAX,
                      1 + (_DS * 63) // INTENSITY_MAX])


def seed_terms(img, x, y):
    """(unary_base, unary_slope, sink_base) from intensity similarity to the
    seed pixel (one table lookup per pixel; same values as the arithmetic)."""
    dsim = np.abs(img - img[y, x]).reshape(-1)
    return tuple(np.take(_TERM_LUT[k], dsim) for k in range(3))


def seed_problem(img, x, y, pairwise, bg, terms=None):
    """Terminal weights from intensity similarity to the seed pixel (the
    seed types of one seed share ``terms``: same arrays, staged once)."""
    height, width = img.shape
    idx = y * width + x
    if idx in bg:
        raise ValueError(f"seed ({x}, {y}) sits on the border")
    base, slope, sink = terms if terms is not None else seed_terms(img, x, y)
    return SeedProblem(width=width, height=height, unary_base=base, unary_slope=slope, sink_base=sink,
                       pairwise=pairwise, fg_seeds=frozenset({idx}), bg_seeds=bg)


def quantize_weights(values, scale: int = 1 << 16) -> np.ndarray:
    """Real-valued weights to integer capacities, round half up at ``scale``
    (harness/synth.py:139-151); negative weights are rejected."""
    if scale < 1:
        raise ValueError("scale must be positive")
    q = np.floor(np.asarray(values, np.float64) * scale + 0.5).astype(np.int64)
    if q.size and int(q.min()) < 0:
        raise ValueError("weights must be non-negative")
    return q


def truth_mask(region, seed_x, seed_y) -> np.ndarray:
    """Flat uint8 mask of the region containing the seed
    (harness/synth.py:102-105)."""
    return (region == region[seed_y, seed_x]).astype(np.uint8).reshape(-1)


@dataclass
class SynthBatch:
    image: np.ndarray
    regions: np.ndarray
    coords: list
    problems: list
    types: tuple = ("A",)

    @property
    def truths(self) -> list:
        """Ground-truth mask per problem (its seed's region), in problem order."""
        return [truth_mask(self.regions, x, y) for (x, y) in self.coords for _ in self.types]


def generate(width, height, seed_rows=1, seed_cols=1, regions=4, noise=10, rng_seed=0,
             types=("A",)) -> SynthBatch:
    """Seed problems of one synthetic image.  types: "A" = reference
    problem_for_seed (border background); "B" = border minus the top row.
    Problems are ordered seed-major, type-minor."""
    rng = np.random.default_rng(rng_seed)
    img, reg = draw_image(width, height, rng, regions, noise)
    pw = contrast_weights(img)
    bgs = {"A": border_pixels(width, height), "B": border_pixels(width, height, top=False)}
    coords = lattice(width, height, seed_rows, seed_cols)
    probs = []
    for (x, y) in coords:
        terms = seed_terms(img, x, y)
        probs += [seed_problem(img, x, y, pw, bgs[t], terms) for t in types]
    return SynthBatch(img, reg, coords, probs, tuple(types))
