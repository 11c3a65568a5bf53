cd /root/repo
python -m paper_1509_06004_b200.build >/dev/null
ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_async$" -c 1 -o gpurun_out/r2_k_async_c2 python scripts/probe.py c2 --reps 1 > gpurun_out/ncu_f2.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_async$" -c 1 -o gpurun_out/r2_k_async_c3 python scripts/probe.py c3 --reps 1 > gpurun_out/ncu_f3.log 2>&1
tail -2 gpurun_out/ncu_f2.log
bash scripts/bench_all.sh r2b
