#!/bin/bash
# run the bench's query step for each built library variant (experiments only)
for so in paper_2101_09441_b200/_lib/libdbl_b200.so paper_2101_09441_b200/_lib/variant_*.so; do
  echo "== $so"
  DBL_LIB_PATH=$PWD/$so timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --box-scale 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,2), 'Gq/s', d['kernel_ms'], 'e2e', round(d['e2e']['value']/1e9,2), 'build', round(d['build']['value_s']*1e3,3), 'ms')"
done
