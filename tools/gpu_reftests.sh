timeout 1100 python tools/ref_tests.py --out gpurun_out/ref_tests.json; echo "ref tests rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
