# pivot prune / wide lean experiment (one GPU)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
for v in "" "DBL_NO_PIVOT_PRUNE=1"; do
  env $v timeout 300 python tools/qbench.py 2>&1 | tail -1
done
for v in "" "DBL_NO_PIVOT_PRUNE=1" "DBL_LEAN_WIDE=1" "DBL_LEAN_WIDE=1 DBL_NO_PIVOT_PRUNE=1"; do
  env $v timeout 600 python tools/cfg5_query.py --label "$v" 2>&1 | tail -1
done
