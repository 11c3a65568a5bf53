#!/bin/bash
# quick GPU check: parity tests + device timings of C2/C3/C4 (probe, 3 reps)
cd "$(dirname "$0")/.."
python -m paper_1509_06004_b200.build >/dev/null || exit 1
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in c2 c3 c4; do timeout 300 python scripts/probe.py $c --reps 4 "$@" | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(d['cfg'], 'med_dev_ms', d['med_dev_ms'], 'push', d['ms_push'], 'bfs', d['ms_bfs'], 'lab', d['ms_labels'], 'cycles', d['cycles'], 'ptp', d['push_tile_passes'], 'btp', d['bfs_tile_passes'], 'bsw', d['bfs_sweeps'])"; done
