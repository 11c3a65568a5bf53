#!/bin/bash
# ncu evidence for round 2 (second session): launch lists (time + DRAM
# bytes) of C5 / C3 / C2 and one --set full capture of each dominant kernel.
cd "$(dirname "$0")/.."
python -m paper_1509_06004_b200.build >/dev/null || exit 1
tag=${1:-r03}
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/${tag}_launches_c5.csv python scripts/probe.py c3 --images 8 --graph 0 --reps 1 > gpurun_out/${tag}_ncu_l5.log 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/${tag}_launches_c3.csv python scripts/probe.py c3 --reps 1 > gpurun_out/${tag}_ncu_l3.log 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/${tag}_launches_c2.csv python scripts/probe.py c2 --reps 1 > gpurun_out/${tag}_ncu_l2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_push -s 8 -c 1 -o gpurun_out/${tag}_k_push_c5 python scripts/probe.py c3 --images 8 --graph 0 --reps 1 > gpurun_out/${tag}_ncu_f5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_bfs_sink -s 40 -c 1 -o gpurun_out/${tag}_k_bfs_c5 python scripts/probe.py c3 --images 8 --graph 0 --reps 1 > gpurun_out/${tag}_ncu_fb5.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_async$" -c 1 -o gpurun_out/${tag}_k_async_c3 python scripts/probe.py c3 --reps 1 > gpurun_out/${tag}_ncu_f3.log 2>&1
ls -la gpurun_out/${tag}_*
