set -x
timeout 300 python tools/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1; echo "rc=$?"; grep -v "^frame\|^ \|omitting" gpurun_out/e2e_probe.log | tail -12
for so in paper_2101_09441_b200/_lib/libdbl_b200.so paper_2101_09441_b200/_lib/variant_*.so; do
  echo "== $so"; DBL_LIB_PATH=$PWD/$so timeout 300 python tools/qbench.py 2>&1 | tail -1
done
