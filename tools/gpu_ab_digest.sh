python tools/digest_ab.py --tag digest > gpurun_out/ab_digest.jsonl 2>&1; echo rc=$?
DBL_LIB_PATH=$PWD/paper_2101_09441_b200/_lib/variant_nodigest.so python tools/digest_ab.py --tag nodigest > gpurun_out/ab_nodigest.jsonl 2>&1; echo rc=$?
cat gpurun_out/ab_digest.jsonl gpurun_out/ab_nodigest.jsonl
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
