set -x
timeout 900 python tools/run_configs.py --cfg 5 --out gpurun_out/cfg5a.json 2>&1 | grep query_qps | cut -c1-300
DBL_LIB_PATH=$PWD/paper_2101_09441_b200/_lib/variant_tall.so timeout 900 python tools/run_configs.py --cfg 5 --out gpurun_out/cfg5b.json 2>&1 | grep query_qps | cut -c1-300
