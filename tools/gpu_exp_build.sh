set -x
L=$PWD/paper_2101_09441_b200/_lib
for v in "DBL_LIB_PATH=$L/variant_any1.so" "" "DBL_LIB_PATH=$L/variant_any8.so"; do
  env $v DBL_TRACE=1 timeout 300 python tools/build_case.py 2>&1 | grep "step" | tail -5
  env $v timeout 300 python tools/qbench.py 2>&1 | tail -1
  env $v DBL_TRACE=1 timeout 600 python tools/cfg5_query.py --nq 100000 --reps 1 2>&1 | grep "step" | tail -5
done
