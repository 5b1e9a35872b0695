#!/bin/bash
for so in paper_2101_09441_b200/_lib/libdbl_b200.so paper_2101_09441_b200/_lib/variant_*.so; do
  echo "== $so"
  DBL_LIB_PATH=$PWD/$so DBL_TRACE=1 python tools/profile_case.py 2>&1 | grep -A4 "build: init frontier" | tail -4
done
