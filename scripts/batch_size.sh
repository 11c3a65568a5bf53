#!/bin/bash
# Device time per CPMC image at 8 / 16 / 32 images per step-synchronous
# batch (the C5 batch-size choice in bench.py).
cd "$(dirname "$0")/.."
for im in 8 16 32; do
  python scripts/probe.py c3 --images $im --reps 3 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print($im, 'images', d['med_dev_ms'], 'ms', round(d['med_dev_ms']/$im,2), 'ms/image', 'cycles', d['cycles'])"
done
