#!/bin/bash
# compute-sanitizer racecheck / synccheck / memcheck over the solver's
# kernels (scripts/sanitize_case.py cases); summaries to gpurun_out/san_*.txt
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
run() {   # tool case limit
    timeout "$3" $CS --tool "$1" --print-limit 20 python scripts/sanitize_case.py "$2" \
        > "gpurun_out/san_$1_$2.txt" 2>&1
    echo "$1 $2 rc=$?" >> gpurun_out/san_summary.txt
    tail -4 "gpurun_out/san_$1_$2.txt" >> gpurun_out/san_summary.txt
}
: > gpurun_out/san_summary.txt
for c in ${CASES:-c1-async c1-sync c1-sync-host comp comp-host wide synth synth-sync stream}; do
    run memcheck $c 300
    run synccheck $c 300
    run racecheck $c 400
done
if [ -z "$CASES" ]; then
run memcheck c3-async 600
run synccheck c3-async 600
fi
