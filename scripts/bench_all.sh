#!/bin/bash
# every bench config + the reference arm, JSON lines into gpurun_out/
cd "$(dirname "$0")/.."
python -m paper_1509_06004_b200.build >/dev/null || exit 1
tag=${1:-r2}
for c in c2 c1 c3 c4 c5; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 > gpurun_out/bench_${tag}_$c.json 2> gpurun_out/bench_${tag}_$c.err
  tail -1 gpurun_out/bench_${tag}_$c.json | cut -c1-250
done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_${tag}_ref.json 2>&1; tail -1 gpurun_out/bench_${tag}_ref.json | cut -c1-200
