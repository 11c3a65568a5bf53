#!/bin/bash
# A/B probe of solver knobs: scripts/ab.sh "<knobs A>" "<knobs B>" ... (each a
# space-separated list of name=value); configs from $CFGS (default: C2, C3
# and an 8-image C5 batch), 5 reps each, median device time
cd "$(dirname "$0")/.."
python -m paper_1509_06004_b200.build >/dev/null || exit 1
CFGS=${CFGS:-"c2;c3;c3 --images 8"}
IFS=';' read -ra CL <<< "$CFGS"
for arm in "$@"; do
  ks=""; for kv in $arm; do ks="$ks --knob $kv"; done
  for cfg in "${CL[@]}"; do
    echo "== [$arm] $cfg"
    timeout 300 python scripts/probe.py $cfg --reps ${REPS:-5} $ks 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print({k:d[k] for k in ('med_dev_ms','flow','cycles','push_tile_passes','bfs_tile_passes','label_tile_passes','ms_push','ms_bfs','ms_labels','ms_async')})"
  done
done
