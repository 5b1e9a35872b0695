set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python tools/qbench.py 2>&1 | tail -1
for v in "" "DBL_LEAN_WIDE=1" "DBL_LIB_PATH=$PWD/paper_2101_09441_b200/_lib/variant_qminb2.so" "DBL_LIB_PATH=$PWD/paper_2101_09441_b200/_lib/variant_qminb1.so"; do
  env $v timeout 600 python tools/cfg5_query.py --label "$v" 2>&1 | tail -1
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_op_read_hit_rate.pct --clock-control none -k regex:"query_fused|label_lean" -c 1 python tools/cfg5_query.py --reps 1 2>&1 | grep -E "query_fused|label_lean|duration|dram__|hit_rate" | tail -4
