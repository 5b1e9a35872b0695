# ncu capture of the cfg5 query kernel (one GPU)
set -x
timeout 600 python tools/cfg5_query.py --label default 2>&1 | tail -1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"query_fused" -c 1 -o gpurun_out/prof_cfg5_pad python tools/cfg5_query.py --reps 1 > gpurun_out/ncu_cfg5.log 2>&1; echo "ncu rc=$?"
tail -2 gpurun_out/ncu_cfg5.log
