#!/bin/bash
# query-kernel experiments on cfg2 (means of 40 flushed batches per run, N runs each)
L=$PWD/paper_2101_09441_b200/_lib
for r in 1 2; do
  for v in "" $EXP_VARIANTS; do
    so=$L/libdbl_b200.so; [ -n "$v" ] && so=$L/variant_$v.so
    echo "== ${v:-base} $(DBL_LIB_PATH=$so timeout 300 python tools/qbench.py --reps 40 2>/dev/null)"
  done
done
