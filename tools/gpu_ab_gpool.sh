# K6 deferred BFS: grid-wide pool for queries past one per warp (product) vs per-CTA queue only
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpool.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpool.log
for r in 1 2 3; do
for v in product gpool0; do
  if [ $v = product ]; then L=""; else L=$PWD/paper_2101_09441_b200/_lib/variant_$v.so; fi
  DBL_LIB_PATH=$L timeout 300 python tools/qbench.py --plain --reps 40 2>&1 | tail -1 | sed "s/^/$v /"
done; done
for v in product gpool0; do
  if [ $v = product ]; then L=""; else L=$PWD/paper_2101_09441_b200/_lib/variant_$v.so; fi
  DBL_LIB_PATH=$L timeout 300 python tools/e2e_probe.py 2>&1 | tail -1 | sed "s/^/$v /"
done
