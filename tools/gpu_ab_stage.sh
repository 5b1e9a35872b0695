timeout 300 python tools/api_batch_probe.py 2>&1 | tail -5 | sed 's/^/staged /'
DBL_LIB_PATH=$PWD/paper_2101_09441_b200/_lib/variant_pipelined.so timeout 300 python tools/api_batch_probe.py 2>&1 | tail -5 | sed 's/^/pipelined /'
nproc
