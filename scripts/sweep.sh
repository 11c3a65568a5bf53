#!/bin/bash
# knob sweep on one config: one JSON line per setting (last of 3 reps)
cfg=${1:-c2}
list=${2:-scripts/sweep_default.txt}
while read -r args; do
  timeout 120 python scripts/probe.py $cfg $args --reps 3 | tail -1
done < "$list"
