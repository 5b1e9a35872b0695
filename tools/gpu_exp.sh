set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/qbench.py 2>&1 | tail -1
DBL_NO_PIVOT=1 timeout 300 python tools/qbench.py 2>&1 | tail -1
DBL_TRACE=1 timeout 300 python tools/qbench.py --reps 3 2>&1 | grep "level\|build:" | tail -24
