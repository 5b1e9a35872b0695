# K6: digest table prefetched into L2 by whole lines at launch (digpf) vs product
for r in 1 2 3; do
for v in product digpf; do
  if [ $v = product ]; then L=""; else L=$PWD/paper_2101_09441_b200/_lib/variant_$v.so; fi
  DBL_LIB_PATH=$L timeout 300 python tools/qbench.py --plain --reps 40 2>&1 | tail -1 | cut -c1-70 | sed "s/^/$v /"
  DBL_LIB_PATH=$L timeout 300 python tools/qbench.py --plain --reps 20 --scale 24 2>&1 | tail -1 | cut -c1-70 | sed "s/^/$v 2^24 /"
done; done
