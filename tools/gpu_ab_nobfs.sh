# K6 split: the full kernel vs the same kernel with the deferred BFS skipped
for r in 1 2; do
for v in product nobfs; do
  if [ $v = product ]; then L=""; else L=$PWD/paper_2101_09441_b200/_lib/variant_$v.so; fi
  DBL_LIB_PATH=$L timeout 300 python tools/qbench.py --plain --reps 40 2>&1 | tail -1 | cut -c1-60 | sed "s/^/$v /"
  DBL_LIB_PATH=$L timeout 300 python tools/qbench.py --plain --reps 40 --novis 2>&1 | tail -1 | cut -c1-60 | sed "s/^/$v novis /"
done; done
