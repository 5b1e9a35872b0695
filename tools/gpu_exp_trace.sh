set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
for v in "" "DBL_NO_CHUNK_LOADS=1" ""; do
  env $v timeout 600 python tools/cfg5_query.py --nq 1000000 --builds 3 2>&1 | tail -1
done
DBL_TRACE=1 timeout 600 python tools/cfg5_query.py --nq 100000 --reps 1 --builds 2 2>&1 | grep "level\|build:" | tail -8
timeout 300 python tools/qbench.py 2>&1 | tail -1
