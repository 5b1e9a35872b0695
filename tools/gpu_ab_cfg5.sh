python tools/cfg5_query.py --label digest > gpurun_out/cfg5_digest.json 2>&1; echo rc=$?
DBL_LIB_PATH=$PWD/paper_2101_09441_b200/_lib/variant_leanwide.so python tools/cfg5_query.py --label leanwide > gpurun_out/cfg5_leanwide.json 2>&1; echo rc=$?
tail -n 2 gpurun_out/cfg5_digest.json gpurun_out/cfg5_leanwide.json
