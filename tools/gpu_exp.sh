set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
DBL_TRACE=1 timeout 300 python tools/qbench.py --reps 3 2>&1 | grep "pivot\|build:" | tail -9
timeout 300 python tools/qbench.py 2>&1 | tail -1
timeout 1500 python tools/run_configs.py --cfg 5 --out gpurun_out/cfg5.json 2>&1 | grep -v "^\[" | tail -2
