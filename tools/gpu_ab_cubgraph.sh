# insert batch: Unique / Flagged / ExclusiveSum replayed as captured graphs too (product) vs direct (cubg0; the sort graph stays)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_cubg.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_cubg.log
for r in 1 2; do
for v in product cubg0; do
  if [ $v = product ]; then L=""; else L=$PWD/paper_2101_09441_b200/_lib/variant_$v.so; fi
  DBL_LIB_PATH=$L timeout 300 python tools/insert_overhead.py 2>&1 | tail -3 | sed "s/^/$v /"
done; done
