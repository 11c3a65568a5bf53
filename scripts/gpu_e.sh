cd $GRAFT_REPO_ROOT
python -m paper_1509_06004_b200.build > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_gputests.log 2>&1; echo "pytest rc $?" >> gpurun_out/t_gputests.log
timeout 900 python bench.py > gpurun_out/t_bench.json 2> gpurun_out/t_bench.err
