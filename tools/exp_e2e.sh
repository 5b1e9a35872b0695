#!/bin/bash
# e2e (pinned host buffers through dbl_query) per library variant
L=$PWD/paper_2101_09441_b200/_lib
for r in 1 2; do
  for v in "" $EXP_VARIANTS; do
    so=$L/libdbl_b200.so; [ -n "$v" ] && so=$L/variant_$v.so
    echo "== ${v:-base} $(DBL_LIB_PATH=$so timeout 300 python tools/e2e_probe.py 2>/dev/null | tail -1)"
  done
done
