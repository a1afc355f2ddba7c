cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/pytest_gpu2.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v1.csv python tools/prof_join.py --count 300000 --reps 1 > gpurun_out/launches_v1.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_join -c 1 -o gpurun_out/prof_join_v1 python tools/prof_join.py --count 300000 --reps 1 > gpurun_out/prof_join_v1.out 2>&1
tail -3 gpurun_out/prof_join_v1.out
