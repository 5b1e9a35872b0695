set -x
for v in "DBL_E2E_ZEROCOPY_IN=1" "DBL_E2E_CHUNKS=4"; do
  env $v DBL_TRACE=0 timeout 300 python tools/e2e_dma.py 2>&1 | tail -2
done
