"""Shared fixtures: golden vectors (produced by the reference, see
tests/golden/make_golden.py) and the ``gpu`` marker."""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built engine")


def _unpack_graphs(z):
    meta, src, snk, nbr = z["meta"], z["src"], z["snk"], z["nbr"]
    out = []
    for (w, h, off) in meta:
        n = int(w) * int(h)
        out.append((int(w), int(h), src[off:off + n], snk[off:off + n],
                    nbr[4 * off:4 * off + 4 * n].reshape(4, n)))
    return out


def load_random(name):
    """[(w, h, src, snk, nbr, flow, labels)] of a random sweep fixture."""
    z = np.load(os.path.join(GOLDEN, name))
    graphs = _unpack_graphs(z)
    flows, labels = z["flows"], z["labels"]
    out, off = [], 0
    for (w, h, s, t, nb), f in zip(graphs, flows):
        out.append((w, h, s, t, nb, int(f), labels[off:off + w * h]))
        off += w * h
    return out


def load_kat():
    with open(os.path.join(GOLDEN, "kat.json")) as f:
        return json.load(f)


def load_composites():
    """[(w, h, src, snk, nbr, record)] of composites_swapped."""
    z = np.load(os.path.join(GOLDEN, "composites_swapped.npz"))
    with open(os.path.join(GOLDEN, "composites_swapped.json")) as f:
        recs = json.load(f)
    return [g + (r,) for g, r in zip(_unpack_graphs(z), recs)]


def load_seed_supergraphs():
    with open(os.path.join(GOLDEN, "seed_supergraphs.json")) as f:
        return json.load(f)


def load_synth(name):
    z = np.load(os.path.join(GOLDEN, name))
    n = int(z["width"]) * int(z["height"])
    labels = np.unpackbits(z["labels_packed"], axis=1, bitorder="little")[:, :n]
    return dict(width=int(z["width"]), height=int(z["height"]), lambdas=tuple(int(v) for v in z["lambdas"]),
                flows=[int(v) for v in z["flows"]], labels=labels,
                sha=str(z["problem_sha256"]),
                composite_flow=int(z["composite_flow"]) if "composite_flow" in z else None)


def problem_digest(p) -> str:
    """sha256 of a SeedProblem's planes and seeds (make_golden.problem_digest)."""
    import hashlib
    h = hashlib.sha256()
    for a in (p.unary_base, p.unary_slope, p.sink_base, p.pairwise):
        h.update(np.ascontiguousarray(a, np.int64).tobytes())
    h.update(np.array(sorted(p.fg_seeds), np.int64).tobytes())
    h.update(np.array(sorted(p.bg_seeds), np.int64).tobytes())
    return h.hexdigest()


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # noqa: BLE001
        return False


@pytest.fixture(scope="session")
def engine():
    """The built native engine on cuda:0 (fails loudly if missing)."""
    from paper_1509_06004_b200 import _native
    return _native.solver_for_thread(0)


def load_scores():
    """Reference scores (harness/bench.py:104-111) of a 96x72, 2x2-seed synth
    batch: per problem flows, foreground counts, exact overlaps."""
    with open(os.path.join(GOLDEN, "scores_96x72_2x2.json")) as f:
        return json.load(f)
