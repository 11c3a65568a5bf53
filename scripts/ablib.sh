#!/bin/bash
# A/B of two builds of the engine: scripts/ablib.sh <libA.so> <libB.so> ...
# (PMF_LIB per arm; configs from $CFGS as in ab.sh), median device time
cd "$(dirname "$0")/.."
python -m paper_1509_06004_b200.build >/dev/null || exit 1
CFGS=${CFGS:-"c2;c3;c3 --images 16"}
IFS=';' read -ra CL <<< "$CFGS"
for r in 1 2; do
for lib in "$@"; do
  for cfg in "${CL[@]}"; do
    echo "== [$lib] $cfg"
    PMF_LIB=$lib timeout 300 python scripts/probe.py $cfg --reps ${REPS:-5} 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print({k:d.get(k) for k in ('med_dev_ms','flow','cycles','push_tile_passes','bfs_tile_passes','ms_push','ms_bfs','ms_labels')})"
  done
done
done
