timeout 300 python tools/insert_overhead.py 2>&1 | tail -3
DBL_LIB_PATH=$PWD/paper_2101_09441_b200/_lib/variant_trace2.so timeout 300 python tools/insert_overhead.py 2>&1 | grep -E "insert:|scale" | tail -14
