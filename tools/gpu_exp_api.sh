set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
./tools/ubench_api
timeout 300 python tools/api_overhead.py 2>&1 | tail -1
DBL_E2E_ZEROCOPY_IN=1 timeout 300 python tools/e2e_dma.py 2>&1 | head -1
timeout 300 python tools/qbench.py 2>&1 | tail -1
