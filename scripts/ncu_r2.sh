#!/bin/bash
# ncu --set full captures of the tile kernels (C3, 4 images, host-driven mode)
cd "$(dirname "$0")/.."
python -m paper_1509_06004_b200.build >/dev/null || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_push -s 8 -c 1 -o gpurun_out/r2_push_c3x4 python scripts/probe.py c3 --images 4 --graph 0 --reps 1 > gpurun_out/ncu_r2a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_bfs_sink -s 8 -c 1 -o gpurun_out/r2_bfs_c3x4 python scripts/probe.py c3 --images 4 --graph 0 --reps 1 > gpurun_out/ncu_r2b.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c3.csv python scripts/probe.py c3 --graph 0 --reps 1 > gpurun_out/ncu_r2c.log 2>&1
ls -la gpurun_out | tail -5
