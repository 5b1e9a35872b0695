set -x
./tools/ubench_query
DBL_NO_FUSED=1 timeout 300 python tools/qbench.py 2>&1 | tail -1
for so in paper_2101_09441_b200/_lib/variant_defer.so paper_2101_09441_b200/_lib/variant_ticket.so; do
  echo "== $so"; DBL_LIB_PATH=$PWD/$so timeout 300 python tools/qbench.py 2>&1 | tail -1
done
