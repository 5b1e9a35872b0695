timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
python tools/digest_ab.py --tag digest > gpurun_out/ab_digest.jsonl 2>&1; echo rc=$?
cat gpurun_out/ab_digest.jsonl
