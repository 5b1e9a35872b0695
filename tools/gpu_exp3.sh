set -x
DBL_BATCHES=4 timeout 300 python tools/insert_case.py 2>&1 | grep batch
DBL_TRACE=1 DBL_BATCHES=3 timeout 300 python tools/insert_case.py 2>&1 | grep -v "build:\|fixpoint levels\|  level" | tail -40
DBL_SCALE=22 DBL_BATCHES=4 timeout 300 python tools/insert_case.py 2>&1 | grep batch
