# K6 device-resident pairs: 1 pair per thread (product) vs 4/8 per thread with
# all digest loads issued ahead, at 4/6/8 resident CTAs per SM
for r in 1 2 3; do
for v in product qdev4 qdev4m6 qdev4m8 qdev8m4; do
  if [ $v = product ]; then L=""; else L=$PWD/paper_2101_09441_b200/_lib/variant_$v.so; fi
  DBL_LIB_PATH=$L timeout 300 python tools/qbench.py --plain --reps 40 2>&1 | tail -1 | sed "s/^/$v /"
done; done
