# e2e zero-copy kernel: digest loads of a thread's 4 pairs issued first (product) vs one pair at a time
for r in 1 2 3; do
for v in product nodpre; do
  if [ $v = product ]; then L=""; else L=$PWD/paper_2101_09441_b200/_lib/variant_$v.so; fi
  DBL_LIB_PATH=$L timeout 300 python tools/e2e_probe.py 2>&1 | tail -1 | sed "s/^/$v /"
done; done
