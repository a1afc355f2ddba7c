cd $GRAFT_REPO_ROOT
for mt in 1 2; do timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_join_umma -s 1 -c 1 -o gpurun_out/b_mt$mt python tools/prof_join.py --reps 1 --mma-tiles $mt > gpurun_out/b_mt$mt.out 2>&1; done
