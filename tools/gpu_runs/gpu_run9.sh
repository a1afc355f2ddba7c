cd $GRAFT_REPO_ROOT
for f in 2 3; do timeout 300 python tools/prof_join.py --count 300000 --reps 2 --filter $f; done
timeout 300 python tools/prof_join.py --reps 2 --filter 2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_join -c 1 -o gpurun_out/prof_join_umma2 python tools/prof_join.py --count 300000 --reps 1 > gpurun_out/prof_join_umma2.out 2>&1
