# K6 grid-size A/B: 1 wave (product) / 2 / 4 waves of resident CTAs
for v in product waves2 waves4 waves4x1024; do
  if [ $v = product ]; then L=""; else L=$PWD/paper_2101_09441_b200/_lib/variant_$v.so; fi
  for r in 1 2; do DBL_LIB_PATH=$L timeout 300 python tools/qbench.py --plain --reps 40 2>&1 | tail -1 | cut -c1-80 | sed "s/^/$v /"; done
done
