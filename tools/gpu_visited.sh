timeout 900 python -m pytest tests/test_visited.py tests/test_serve.py -x -q 2>&1 | tail -15
timeout 1100 python tools/ref_tests.py --out gpurun_out/ref_tests.json; echo "ref tests rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
