set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu.log
L=$PWD/paper_2101_09441_b200/_lib
for v in "" "DBL_LIB_PATH=$L/variant_qnodefer.so" ""; do
  env $v timeout 600 python tools/cfg5_query.py 2>&1 | tail -1
done
