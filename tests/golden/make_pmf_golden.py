"""Golden ``.pmf`` batch from the REFERENCE writer (harness/problemio.py).

    python tests/golden/make_pmf_golden.py

Writes batch_small.pmf (+ its .json sidecar): the reference's synthetic
generator's problems and truth masks for a 24x18 image with 2x2 seed
points and both seed types (harness/synth.py:108), through
``write_problem_file`` with a small metadata dict.  Run in the build
container (reference mounted at /root/reference).
"""

from __future__ import annotations

import os
import sys

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from pmflow.harness.config import BenchConfig  # noqa: E402
from pmflow.harness.problemio import write_problem_file  # noqa: E402
from pmflow.harness.synth import generate_batch  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "batch_small.pmf")


def main():
    cfg = BenchConfig(width=24, height=18, seed_rows=2, seed_cols=2, rng_seed=4)
    meta, probs, truths = generate_batch(cfg)
    write_problem_file(OUT, probs, truths, meta=meta)
    print(OUT, len(probs), "problems")


if __name__ == "__main__":
    main()
