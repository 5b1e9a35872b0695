set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
DBL_BATCHES=5 timeout 300 python tools/insert_case.py 2>&1 | grep batch
DBL_SCALE=22 DBL_BATCHES=5 timeout 300 python tools/insert_case.py 2>&1 | grep batch
