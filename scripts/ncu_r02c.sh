#!/bin/bash
# ncu evidence for round 2 (third session): launch lists (time + DRAM bytes)
# of C5 (32 images, device-synthesised and host-staged), C3, C2 and one
# --set full capture of each dominant kernel plus the synthesis kernels.
cd "$(dirname "$0")/.."
python -m paper_1509_06004_b200.build >/dev/null || exit 1
tag=${1:-r02c}
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
P="python scripts/probe.py"
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/${tag}_launches_c5.csv $P c3 --images 32 --graph 0 --reps 1 > gpurun_out/${tag}_l5.log 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/${tag}_launches_c5s.csv $P c3 --images 32 --synth --graph 0 --reps 1 > gpurun_out/${tag}_l5s.log 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/${tag}_launches_c3.csv $P c3 --reps 1 > gpurun_out/${tag}_l3.log 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/${tag}_launches_c2.csv $P c2 --reps 1 > gpurun_out/${tag}_l2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_push -s 8 -c 1 -o gpurun_out/${tag}_k_push_c5 $P c3 --images 32 --graph 0 --reps 1 > gpurun_out/${tag}_f5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_bfs_sink -s 40 -c 1 -o gpurun_out/${tag}_k_bfs_c5 $P c3 --images 32 --graph 0 --reps 1 > gpurun_out/${tag}_fb5.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_async$" -c 1 -o gpurun_out/${tag}_k_async_c3 $P c3 --reps 1 > gpurun_out/${tag}_f3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_synth|k_pack_bits|k_seed_masks" -c 4 -o gpurun_out/${tag}_k_synth_c5 $P c3 --images 32 --synth --graph 0 --reps 1 > gpurun_out/${tag}_fs5.log 2>&1
ls -la gpurun_out/${tag}_*
