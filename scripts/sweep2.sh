#!/bin/bash
# knob sweep: for each line of $1, C2 and C3 device time (probe, 3 reps)
cd "$(dirname "$0")/.."
python -m paper_1509_06004_b200.build >/dev/null || exit 1
while read -r args; do
  for c in ${CFGS:-c2 c3}; do
    timeout 120 python scripts/probe.py $c --reps 3 $args | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(d['cfg'], '[$args]', 'dev', d['med_dev_ms'], 'push', d['ms_push'], 'bfs', d['ms_bfs'], 'cyc', d['cycles'], 'ptp', d['push_tile_passes'], 'btp', d['bfs_tile_passes'], 'bsw', d['bfs_sweeps'], 'scan', d.get('scan_tile_passes'), 'lab', d['label_tile_passes'])" || echo "$c [$args] FAILED"
  done
done < "$1"
