# profiling runner (used via gpurun): fused query kernel under ncu with and without ncu's own cache flush,
# plus the per-level fixpoint trace
set -x
DBL_TRACE=1 timeout 300 python tools/qbench.py --reps 3 > gpurun_out/trace.log 2>&1; echo "trace rc=$?"; grep -A12 "fixpoint levels" gpurun_out/trace.log | head -30; grep "\[dbl\]" gpurun_out/trace.log | head -60
timeout 600 ncu --set full --clock-control none --import-source on -k regex:query_fused -c 3 -o gpurun_out/q_flush python tools/qbench.py --reps 3 > gpurun_out/ncu_q1.log 2>&1; echo "ncu1 rc=$?"
timeout 600 ncu --set full --clock-control none --cache-control none --import-source on -k regex:query_fused -c 3 -o gpurun_out/q_noflush python tools/qbench.py --reps 3 > gpurun_out/ncu_q2.log 2>&1; echo "ncu2 rc=$?"
