# ncu capture of the cfg5 query kernels (one GPU)
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"query_fused|label_lean|bfs_warp" -c 3 -o gpurun_out/prof_cfg5_fused python tools/cfg5_query.py --reps 1 > gpurun_out/ncu_cfg5a.log 2>&1; echo "ncu a rc=$?"
tail -3 gpurun_out/ncu_cfg5a.log
DBL_LEAN_WIDE=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"query_fused|label_lean|bfs_warp" -c 3 -o gpurun_out/prof_cfg5_lean python tools/cfg5_query.py --reps 1 > gpurun_out/ncu_cfg5b.log 2>&1; echo "ncu b rc=$?"
tail -3 gpurun_out/ncu_cfg5b.log
