# Same-box A/B of the label build: variant_base.so (tools/build_rev.py REV base) vs the tree's library.
# AB_CASES="20_8_64 26_16_256" (scale_edgefactor_k) overrides the default cases.
L=$PWD/paper_2101_09441_b200/_lib
for r in 1 2; do
for v in base cur; do
  if [ $v = base ]; then export DBL_LIB_PATH=$L/variant_base.so; else unset DBL_LIB_PATH; fi
  for sc in ${AB_CASES:-20_8_64 22_8_64 24_8_64 26_16_256}; do set -- ${sc//_/ }
    python tools/build_profile.py --scale $1 --ef $2 --k $3 --reps 10 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$v', d['scale'], d['k'], round(d['mean_ms'],4), round(d['min_ms'],4))"
  done
done; done
