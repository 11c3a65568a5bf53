#!/bin/bash
# Round-end evidence: ncu launch lists + --set full captures (scripts/ncu_r02c.sh),
# every bench config and the reference arm; outputs gpurun_out/<tag>_*.
cd "$(dirname "$0")/.."
tag=${1:-r02d}
python -m paper_1509_06004_b200.build > /dev/null || exit 1
timeout 1500 bash scripts/ncu_r02c.sh $tag > gpurun_out/${tag}_ncu.log 2>&1
timeout 900 python scripts/memguard.py --floor 24 -- python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
for c in c3 c2 c1 c4; do
  timeout 600 python bench.py --config $c --no-secondary > gpurun_out/${tag}_bench_$c.json 2>> gpurun_out/${tag}_bench.err
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${tag}_bench_ref.json 2>> gpurun_out/${tag}_bench.err
