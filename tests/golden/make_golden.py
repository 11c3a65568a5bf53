"""Generate golden vectors by running the REFERENCE package (pmflow).

Run in the build container, where the reference is mounted read-only at
/root/reference:

    python tests/golden/make_golden.py [--big]

The outputs (small .npz / .json files next to this script) are committed, so
the GPU box -- which has no /root/reference -- can check parity against them.
Every vector comes from the reference's own public API:
``maxflow_pushrelabel`` (solvers.py:188), ``solve_composite``
(supergraph.py:190), ``split`` (:157), ``build_seed_supergraph`` (:227),
``solve_schedule_sequential`` (parametric.py:180), ``generate_batch``
(harness/synth.py:108).  ``--big`` adds the C2 (500x375, 20 lambda)
per-lambda fixture, which takes ~70 s of reference CPU time.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))

from conftest import make_grid, random_grid  # noqa: E402  (reference test helpers)
from pmflow.grid import CAP_MAX  # noqa: E402
from pmflow.harness.config import BenchConfig  # noqa: E402
from pmflow.harness.synth import generate_batch  # noqa: E402
from pmflow.parametric import LambdaSchedule, SeedProblem, solve_schedule_sequential  # noqa: E402
from pmflow.solvers import maxflow_pushrelabel  # noqa: E402
from pmflow.supergraph import (apply_swap, build_seed_supergraph, join,  # noqa: E402
                               solve_composite, split)

OUT = os.path.dirname(os.path.abspath(__file__))
L20 = (2, 3, 4, 5, 7, 9, 12, 16, 22, 30, 40, 54, 73, 99, 134, 181, 244, 329, 444, 600)


def pack_graphs(graphs):
    """Variable-size graphs -> flat arrays + per-graph (w, h, offset)."""
    meta, src, snk, nbr = [], [], [], []
    off = 0
    for g in graphs:
        meta.append((g.width, g.height, off))
        src.append(g.src_cap)
        snk.append(g.snk_cap)
        nbr.append(g.nbr_cap.reshape(-1))
        off += g.n
    return dict(meta=np.array(meta, np.int64), src=np.concatenate(src),
                snk=np.concatenate(snk), nbr=np.concatenate(nbr))


def problem_digest(p: SeedProblem) -> str:
    h = hashlib.sha256()
    for a in (p.unary_base, p.unary_slope, p.sink_base, p.pairwise):
        h.update(np.ascontiguousarray(a, np.int64).tobytes())
    h.update(np.array(sorted(p.fg_seeds), np.int64).tobytes())
    h.update(np.array(sorted(p.bg_seeds), np.int64).tobytes())
    return h.hexdigest()


def kat():
    """Hand fixtures of tests/test_solvers.py:19-62 and SPEC examples."""
    cases = {
        "single_pixel_zero": make_grid(1, 1),
        "two_pixel_chain": make_grid(2, 1, src=[5, 0], snk=[0, 3], right=[2, 0], left=[0, 2]),
        "two_by_two_diagonal": make_grid(2, 2, src=[9, 0, 0, 0], snk=[0, 0, 0, 9],
                                         left=[0, 1, 0, 1], right=[1, 0, 1, 0],
                                         up=[0, 0, 1, 1], down=[1, 1, 0, 0]),
        "zero_3x3": make_grid(3, 3),
        "unreachable_foreground": make_grid(2, 1, src=[5, 0], snk=[0, 0], right=[2, 0], left=[0, 2]),
        "seed_cap_max": make_grid(3, 1, src=[CAP_MAX, 0, 1], snk=[0, 4, 0], right=[3, 1, 0],
                                  left=[0, 3, 1]),
    }
    out = {}
    for name, g in cases.items():
        r = maxflow_pushrelabel(g)
        out[name] = dict(width=g.width, height=g.height, src=g.src_cap.tolist(),
                         snk=g.snk_cap.tolist(), nbr=g.nbr_cap.tolist(), flow=r.flow,
                         labels=r.labels.tolist())
    with open(os.path.join(OUT, "kat.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


def random_sweep(name, seed, count, max_side, cap_hi):
    rng = np.random.default_rng(seed)
    graphs = [random_grid(rng, max_side=max_side, cap_hi=cap_hi) for _ in range(count)]
    flows, labels = [], []
    for g in graphs:
        r = maxflow_pushrelabel(g)
        flows.append(r.flow)
        labels.append(r.labels)
    np.savez_compressed(os.path.join(OUT, name), flows=np.array(flows, np.int64),
                        labels=np.concatenate(labels), **pack_graphs(graphs))


def composite_sweep(name, seed, count):
    """Composite-level labels with random swap flags and padding: the pins of
    test_rpc.py:28-35 / test_supergraph.py:189-204 for solve_composite's
    swapped-span semantics (supergraph.py:201-206)."""
    rng = np.random.default_rng(seed)
    records = []
    comps = []
    for _ in range(count):
        k = int(rng.integers(1, 5))
        graphs = [random_grid(rng, max_side=6) for _ in range(k)]
        flags = [bool(rng.integers(0, 2)) for _ in range(k)]
        embedded = [apply_swap(g) if f else g for g, f in zip(graphs, flags)]
        composite, layout = join(embedded, swapped=flags, pad=True)
        cut = solve_composite(composite, layout)
        parts = split(layout, cut, graphs)
        comps.append(composite)
        records.append(dict(
            segments=[[s.offset, s.width, int(s.swapped)] for s in layout.segments],
            originals=[[g.width, g.height] for g in graphs],
            flow=cut.flow, part_flows=[p.flow for p in parts]))
        records[-1]["labels"] = cut.labels.tolist()
    np.savez_compressed(os.path.join(OUT, name), **pack_graphs(comps))
    with open(os.path.join(OUT, name + ".json"), "w") as f:
        json.dump(records, f)


def seed_supergraph_cases():
    """build_seed_supergraph + solve_composite + split for swap modes."""
    rng = np.random.default_rng(70)
    out = []
    for mode in ("auto", "on", "off"):
        for trial in range(3):
            w, h = int(rng.integers(3, 7)), int(rng.integers(3, 7))
            n = w * h
            probs = []
            for _ in range(int(rng.integers(1, 4))):
                pw = np.zeros((4, h, w), np.int64)
                pw[1, :, :-1] = rng.integers(0, 5, (h, w - 1))
                pw[0, :, 1:] = rng.integers(0, 5, (h, w - 1))
                pw[3, :-1, :] = rng.integers(0, 5, (h - 1, w))
                pw[2, 1:, :] = rng.integers(0, 5, (h - 1, w))
                fg = int(rng.integers(0, n))
                bg = (fg + 1 + int(rng.integers(0, n - 1))) % n
                probs.append(SeedProblem(width=w, height=h,
                                         unary_base=rng.integers(0, 6, n),
                                         unary_slope=rng.integers(0, 3, n),
                                         sink_base=rng.integers(0, 25, n),
                                         pairwise=pw.reshape(4, n),
                                         fg_seeds=frozenset({fg}), bg_seeds=frozenset({bg})))
            sched = LambdaSchedule((0, 1, 3, 8, 20))
            comp, layout, originals = build_seed_supergraph(probs, sched, mode)
            cut = solve_composite(comp, layout)
            parts = split(layout, cut, originals)
            out.append(dict(
                mode=mode, width=w, height=h, lambdas=list(sched.values),
                problems=[dict(base=p.unary_base.tolist(), slope=p.unary_slope.tolist(),
                               sink=p.sink_base.tolist(), pairwise=p.pairwise.tolist(),
                               fg=sorted(p.fg_seeds), bg=sorted(p.bg_seeds)) for p in probs],
                swapped=[s.swapped for s in layout.segments],
                composite_width=comp.width, composite_flow=cut.flow,
                composite_labels=cut.labels.tolist(),
                flows=[p.flow for p in parts], labels=[p.labels.tolist() for p in parts]))
    with open(os.path.join(OUT, "seed_supergraphs.json"), "w") as f:
        json.dump(out, f)


def synth_config(name, width, height, lambdas, rows=1, cols=1, rng_seed=0, composite=False):
    """Per-lambda reference cuts on a synth problem (labels bit-packed)."""
    cfg = BenchConfig(width=width, height=height, seed_rows=rows, seed_cols=cols,
                      rng_seed=rng_seed)
    _, problems, _ = generate_batch(cfg)
    p = problems[0]
    seq = solve_schedule_sequential(p, LambdaSchedule(lambdas))
    rec = dict(width=width, height=height, rng_seed=rng_seed, lambdas=list(lambdas),
               problem_sha256=problem_digest(p),
               flows=np.array([c.flow for c in seq.cuts], np.int64),
               labels_packed=np.packbits(np.stack([c.labels for c in seq.cuts]), axis=1,
                                         bitorder="little"))
    if composite:
        comp, layout, originals = build_seed_supergraph([p], LambdaSchedule(lambdas), "auto")
        cut = solve_composite(comp, layout)
        parts = split(layout, cut, originals)
        assert [q.flow for q in parts] == rec["flows"].tolist()
        rec["composite_flow"] = np.int64(cut.flow)
    np.savez_compressed(os.path.join(OUT, name), **rec)


def synth_scores(name, width, height, lambdas, rows=1, cols=1, rng_seed=0):
    """Reference scoring of per-lambda cuts (harness/bench.py:104-111):
    foreground counts and exact overlaps with the truth masks, per problem."""
    from pmflow.harness.bench import overlap
    cfg = BenchConfig(width=width, height=height, seed_rows=rows, seed_cols=cols,
                      rng_seed=rng_seed)
    _, problems, truths = generate_batch(cfg)
    recs = []
    for p, t in zip(problems, truths):
        seq = solve_schedule_sequential(p, LambdaSchedule(lambdas))
        ov = [overlap(c.labels, t) for c in seq.cuts]
        recs.append(dict(problem_sha256=problem_digest(p),
                         truth_sha256=hashlib.sha256(np.asarray(t, np.uint8).tobytes()).hexdigest(),
                         flows=[c.flow for c in seq.cuts],
                         foreground=[int(c.labels.sum()) for c in seq.cuts],
                         overlap=[[o.numerator, o.denominator] for o in ov]))
    with open(os.path.join(OUT, name), "w") as f:
        json.dump(dict(width=width, height=height, rows=rows, cols=cols, rng_seed=rng_seed,
                       lambdas=list(lambdas), problems=recs), f)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--only-scores", action="store_true")
    args = ap.parse_args()
    if args.only_scores:
        synth_scores("scores_96x72_2x2.json", 96, 72, LambdaSchedule.default().values, rows=2, cols=2,
                     rng_seed=5)
        return
    kat()
    random_sweep("random_8x8_seed101.npz", 101, 500, 8, 10)     # test_acceptance.py:34-46
    random_sweep("random_3x3_seed102.npz", 102, 100, 3, 10)     # :49-60
    composite_sweep("composites_swapped", 34, 40)
    seed_supergraph_cases()
    synth_config("c1_160x120.npz", 160, 120, LambdaSchedule.default().values, composite=True)
    synth_scores("scores_96x72_2x2.json", 96, 72, LambdaSchedule.default().values, rows=2, cols=2, rng_seed=5)
    if args.big:
        synth_config("c2_500x375.npz", 500, 375, L20)


if __name__ == "__main__":
    main()
