#!/bin/bash
# ncu evidence for the round-2 engine: launch lists (time + DRAM bytes) and
# one --set full capture of each dominant kernel
cd "$(dirname "$0")/.."
python -m paper_1509_06004_b200.build >/dev/null || exit 1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2_launches_c2.csv python scripts/probe.py c2 --reps 1 > gpurun_out/ncu_l2.log 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2_launches_c3.csv python scripts/probe.py c3 --reps 1 > gpurun_out/ncu_l3.log 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2_launches_c5.csv python scripts/probe.py c3 --images 8 --graph 0 --reps 1 > gpurun_out/ncu_l5.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_async$" -c 1 -o gpurun_out/r2_k_async_c2 python scripts/probe.py c2 --reps 1 > gpurun_out/ncu_f2.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_async$" -c 1 -o gpurun_out/r2_k_async_c3 python scripts/probe.py c3 --reps 1 > gpurun_out/ncu_f3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_push -s 8 -c 1 -o gpurun_out/r2_k_push_c5 python scripts/probe.py c3 --images 8 --graph 0 --reps 1 > gpurun_out/ncu_f5.log 2>&1
ls -la gpurun_out/*.ncu-rep gpurun_out/r2_launches*
