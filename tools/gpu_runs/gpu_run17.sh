cd $GRAFT_REPO_ROOT
(cd old_r18 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_join_umma -s 1 -c 1 -o ../gpurun_out/cmp_old python tools/prof_join.py --reps 1 > ../gpurun_out/cmp_old.out 2>&1)
for mt in 1 2; do timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_join_umma -s 1 -c 1 -o gpurun_out/cmp_mt$mt python tools/prof_join.py --reps 1 --mma-tiles $mt > gpurun_out/cmp_mt$mt.out 2>&1; done
tail -2 gpurun_out/cmp_*.out
