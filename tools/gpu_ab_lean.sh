# K6 CTA size A/B (256 product / 512 / 1024): cfg2 batch kernel and e2e
for v in product lean512 lean1024; do
  if [ $v = product ]; then L=""; else L=$PWD/paper_2101_09441_b200/_lib/variant_$v.so; fi
  for r in 1 2; do DBL_LIB_PATH=$L timeout 300 python tools/qbench.py --plain --reps 40 2>&1 | tail -1 | sed "s/^/$v /"; done
  DBL_LIB_PATH=$L timeout 300 python tools/e2e_probe.py 2>&1 | tail -2 | sed "s/^/$v /"
done
