timeout 1100 python tools/ref_tests.py --out gpurun_out/ref_tests.json; echo "ref tests rc=$?"
timeout 900 python -m pytest tests/test_cli.py tests/test_snapshot.py tests/test_gpu_extras.py -x -q > gpurun_out/pytest_cli.log 2>&1; echo "cli rc=$?"; tail -3 gpurun_out/pytest_cli.log
