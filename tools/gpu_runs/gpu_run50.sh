cd $GRAFT_REPO_ROOT
timeout 600 python tools/prof_join.py --workload songs90 --reps 2 --filter 1 2>&1 | tail -1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_join32 -s 1 -c 1 -o gpurun_out/prof_songs005 python tools/prof_join.py --workload songs90 --reps 1 --filter 1 > gpurun_out/prof_songs005.out 2>&1; tail -1 gpurun_out/prof_songs005.out
