set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
for v in ""; do
  env $v timeout 600 python tools/cfg5_query.py --label "$v" 2>&1 | tail -1
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_op_read_hit_rate.pct,lts__t_requests_srcunit_tex_op_read.sum --clock-control none -k regex:"query_quad" -c 1 python tools/cfg5_query.py --reps 1 2>&1 | grep -E "query_quad|duration|dram__|hit_rate|requests" | tail -5
