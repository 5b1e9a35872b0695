set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for r in 1 2; do
for so in paper_2101_09441_b200/_lib/libdbl_b200.so paper_2101_09441_b200/_lib/variant_*.so; do
  echo "== $so"; DBL_LIB_PATH=$PWD/$so timeout 300 python tools/qbench.py --reps 60 2>&1 | tail -1
done
done
