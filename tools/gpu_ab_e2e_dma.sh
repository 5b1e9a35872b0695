# e2e from pinned host buffers: zero-copy kernel (product) vs the chunked copy
# pipeline (copy engine H2D per chunk, kernel per chunk, D2H per chunk)
for r in 1 2; do
for v in product dma17 dma18 dma19; do
  if [ $v = product ]; then L=""; else L=$PWD/paper_2101_09441_b200/_lib/variant_$v.so; fi
  DBL_LIB_PATH=$L timeout 300 python tools/e2e_probe.py 2>&1 | tail -1 | sed "s/^/$v /"
done; done
