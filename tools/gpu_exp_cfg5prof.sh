# ncu captures for cfg5 (one GPU): the wide query kernel and the build kernels
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"query_quad|reach_kernel|fixpoint_kernel|prep_kernel" -c 5 -o gpurun_out/prof_cfg5_r01 python tools/cfg5_query.py --reps 1 > gpurun_out/ncu_cfg5.log 2>&1; echo "ncu rc=$?"
tail -2 gpurun_out/ncu_cfg5.log
